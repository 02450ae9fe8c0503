"""Build and run tools/ubench.cu (FP32 FFMA, MUFU ex2, SHFL, LDS.128, RED throughput and HBM
copy on this GPU).  Writes the JSON line to profiles/<name>.json.

    python tools/ubench.py [--out profiles/r1_ubench.json]
"""
import argparse
import json
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)


def main(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "r1_ubench.json"))
    a = ap.parse_args(argv)
    exe = os.path.join(HERE, "ubench")
    subprocess.check_call(["/usr/local/cuda/bin/nvcc", "-O3", "-gencode", "arch=compute_100a,code=sm_100a",
                           "-std=c++17", "-o", exe, os.path.join(HERE, "ubench.cu")])
    res = json.loads(subprocess.check_output([exe]).decode())
    clk = subprocess.run(["nvidia-smi", "--query-gpu=clocks.sm,clocks.max.sm", "--format=csv,noheader,nounits"],
                         capture_output=True, text=True).stdout.strip()
    res["nvidia_smi_clocks_after"] = clk
    os.makedirs(os.path.dirname(a.out), exist_ok=True)
    with open(a.out, "w") as f:
        json.dump(res, f, indent=1)
    print(json.dumps(res))


if __name__ == "__main__":
    sys.exit(main())
