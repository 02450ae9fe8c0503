#!/bin/bash
# A/B timing of build variants on one B200 (run from the repo root under gpurun):
#   tools/variant_bench.sh "<label>=<GS_NVCC_EXTRA flags>" ... [-- bench args]
# Each variant is rebuilt (--force) and timed with a short bench; one line per variant with
# the step and per-stage device times goes to gpurun_out/variants.txt.
args=()
vars=()
while [ $# -gt 0 ]; do
  if [ "$1" = "--" ]; then shift; args=("$@"); break; fi
  vars+=("$1"); shift
done
for v in "${vars[@]}"; do
  label="${v%%=*}"; flags="${v#*=}"
  GS_NVCC_EXTRA="$flags" python -m paper_2409_06765_b200.build --force > /dev/null || { echo "$label build failed" >> gpurun_out/variants.txt; continue; }
  timeout 600 python bench.py --no-cpu-baseline --no-e2e --no-strong --no-variants --steps 10 "${args[@]}" > gpurun_out/v_$label.json 2> gpurun_out/v_$label.err
  python - "$label" "gpurun_out/v_$label.json" "${args[*]}" >> gpurun_out/variants.txt <<'PY'
import json, sys
lab, f, a = sys.argv[1], sys.argv[2], sys.argv[3]
try:
    d = json.loads(open(f).read().strip().splitlines()[-1])
except Exception as e:
    print(f"{lab:14s} [{a}] FAILED {e}"); sys.exit()
st = " ".join(f"{k}={v['ms']:.4f}" for k, v in d["stages"].items())
print(f"{lab:14s} [{a}] {d['value']:8.1f} {d['unit']} step {d['ms_per_step']:.4f} ms  {st}")
PY
done
python -m paper_2409_06765_b200.build --force > /dev/null
