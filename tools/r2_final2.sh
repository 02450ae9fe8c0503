# Round-2 final measurement set (after the packed FP32x2 change) on one B200, run from the repo
# root under gpurun; compute-sanitizer is closed on this pool, so that leg is dropped.
set -x
mkdir -p gpurun_out
nvidia-smi -q -d CLOCK | head -30 > gpurun_out/f_clocks.txt
timeout 900 python bench.py > gpurun_out/f_bench.json 2> gpurun_out/f_bench.err
: > gpurun_out/f_bench_configs.jsonl
for c in "batch3m 8" "large6m 4" "aa_packed1m 4"; do set -- $c
  timeout 900 python bench.py --config $1 --views-per-gpu $2 --no-cpu-baseline --no-strong --steps 10 >> gpurun_out/f_bench_configs.jsonl 2>> gpurun_out/f_bench.err
done
timeout 600 python bench.py --shard gaussians --views-per-gpu 4 --steps 10 > gpurun_out/f_bench_gshard.json 2>> gpurun_out/f_bench.err
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:^k_ --launch-skip 32 --launch-count 64 --csv --log-file gpurun_out/f_launches.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-strong --no-variants --eager > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:^k_ --launch-skip 32 --launch-count 32 -o gpurun_out/f_full python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-strong --no-variants --eager > /dev/null 2>&1
ncu --set full --clock-control none -k regex:"k_raster_bwd|k_project_bwd" --launch-skip 2 --launch-count 2 -o gpurun_out/f_c2_k78 python bench.py --config batch3m --views-per-gpu 8 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --no-strong --no-variants --eager > /dev/null 2>&1
timeout 900 python bench.py --impl reference --steps 1 --warmup 3 > gpurun_out/f_reference.json 2>> gpurun_out/f_bench.err
GS_PARITY_REPORT=gpurun_out/f_parity_report.jsonl timeout 1200 python -m pytest tests -m gpu -q 2>&1 | tail -5 > gpurun_out/f_gputest.txt
ls -la gpurun_out
