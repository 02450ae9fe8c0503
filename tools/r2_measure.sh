# Round-2 measurement set on one B200 (run from the repo root under gpurun).
set -x
timeout 900 python bench.py > gpurun_out/r2_bench.json 2> gpurun_out/r2_bench.err
: > gpurun_out/r2_bench_configs.jsonl
for c in "batch3m 8" "large6m 4" "aa_packed1m 4"; do set -- $c
  timeout 900 python bench.py --config $1 --views-per-gpu $2 --no-cpu-baseline --no-strong --steps 10 >> gpurun_out/r2_bench_configs.jsonl 2>> gpurun_out/r2_bench.err
done
timeout 600 python bench.py --shard gaussians --views-per-gpu 4 --steps 10 > gpurun_out/r2_bench_gshard.json 2>> gpurun_out/r2_bench.err
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:^k_ --launch-skip 31 --launch-count 31 --csv --log-file gpurun_out/r2_launches.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-strong --no-variants --eager > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:^k_ --launch-skip 31 --launch-count 31 -o gpurun_out/r2_full python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-strong --no-variants --eager > /dev/null 2>&1
timeout 900 python bench.py --impl reference --steps 1 --warmup 3 > gpurun_out/r2_reference.json 2>> gpurun_out/r2_bench.err
ls -la gpurun_out
