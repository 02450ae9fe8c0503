"""Summarise ncu captures for profiles/ (run here, on the CPU box, on files gpurun
brought back in gpurun_out/).

  python tools/ncu_summary.py launches <launches.csv> > profiles/rN_launches.txt
  python tools/ncu_summary.py full <report.ncu-rep> [--traffic profiles/traffic.json --workload garden1m/views1] > profiles/rN_full.txt
"""
import csv
import json
import os
import re
import subprocess
import sys

STAGE_OF = {"k_project_fwd": "project", "k_raster_fwd": "raster_fwd", "k_raster_bwd": "raster_bwd",
            "k_project_bwd": "project_bwd", "k_zero4": "raster_bwd", "k_tile_work": "raster_bwd",
            "k_tile_order": "raster_bwd"}
ISECT = ("k_vis_", "k_scan_blocksums", "k_radix_", "k_tiles_", "k_ranges", "k_packed_items", "k_keys64")


def stage_of(name):
    if name in STAGE_OF:
        return STAGE_OF[name]
    return "isect" if name.startswith(ISECT) else None
KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "smsp__inst_executed.sum",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "smsp__thread_inst_executed_per_inst_executed.ratio", "launch__registers_per_thread",
        "launch__occupancy_limit_registers", "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", "lts__t_sectors.sum",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "l1tex__t_requests_pipe_lsu_mem_global_op_red.sum",
        "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_wait_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_not_selected_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_lg_throttle_per_issue_active.ratio"]


def short(n):
    m = re.search(r"(k_\w+)", n)
    return m.group(1) if m else n[:40]


def launches(path):
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hi]
    ki, mi, vi, ii = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("ID")
    ks = [(int(r[ii]), r[ki], float(r[vi].replace(",", ""))) for r in rows[hi + 1:]
          if len(r) > vi and r[mi] == "gpu__time_duration.sum"]
    starts = [j for j, k in enumerate(ks) if "k_project_fwd" in k[1]]
    st = starts[-1]
    if st > 0 and "k_zero4" in ks[st - 1][1]:   # the side-stream zero-fill forked at the step start
        st -= 1
    end = next(j for j in range(st, len(ks)) if "k_project_bwd" in ks[j][1])
    step = ks[st:end + 1]
    tot = sum(v for _, _, v in step)
    print("# ncu --metrics gpu__time_duration.sum --clock-control none (cold, serialised launches)")
    print(f"# last full step: {len(step)} launches of libgsplat_b200, sum {tot / 1e3:.1f} us")
    for i, n, v in step:
        print(f"{i:5d}  {short(n):24s} {v / 1e3:9.1f} us  {100 * v / tot:5.1f} %")
    agg = {}
    for _, n, v in step:
        agg[short(n)] = agg.get(short(n), 0) + v
    print("# by kernel")
    for k, v in sorted(agg.items(), key=lambda x: -x[1]):
        print(f"   {k:24s} {v / 1e3:9.1f} us  {100 * v / tot:5.1f} %")


def full(path, traffic_out=None, workload=None):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    h, u = rows[0], rows[1]
    traffic = {}
    print(f"# ncu --set full --clock-control none summary of {path.split('/')[-1]}")
    for r in rows[2:]:
        name = short(r[h.index("Kernel Name")])
        print(f"== {name}")
        for k in KEYS:
            if k in h and r[h.index(k)]:
                print(f"   {k:78s} {r[h.index(k)]} {u[h.index(k)]}")
        st = stage_of(name)
        if st:
            rd = float(r[h.index("dram__bytes_read.sum")].replace(",", ""))
            wr = float(r[h.index("dram__bytes_write.sum")].replace(",", ""))
            mult = {"Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "byte": 1.0}
            b = rd * mult[u[h.index("dram__bytes_read.sum")]] + wr * mult[u[h.index("dram__bytes_write.sum")]]
            t = traffic.setdefault(st, {"kernels": [], "dram_bytes_per_launch": 0.0, "source": path.split("/")[-1]})
            t["kernels"].append(name)
            t["dram_bytes_per_launch"] += b   # the stage's kernels of one step summed
    if traffic_out:
        # keyed by the bench workload the capture was taken on (bench.traffic_key)
        allw = json.load(open(traffic_out)) if os.path.exists(traffic_out) else {}
        allw[workload] = traffic
        json.dump(allw, open(traffic_out, "w"), indent=1)


if __name__ == "__main__":
    if sys.argv[1] == "launches":
        launches(sys.argv[2])
    else:
        tr = sys.argv[sys.argv.index("--traffic") + 1] if "--traffic" in sys.argv else None
        wl = sys.argv[sys.argv.index("--workload") + 1] if "--workload" in sys.argv else None
        if tr and not wl:
            sys.exit("--traffic needs --workload (the bench workload key, e.g. garden1m/views1)")
        full(sys.argv[2], tr, wl)
