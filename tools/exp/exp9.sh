mkdir -p gpurun_out
: > gpurun_out/variants.txt
tools/variant_bench.sh "prep="
tools/variant_bench.sh "prep=" -- --config batch3m --views-per-gpu 8
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -4 > gpurun_out/exp9_tests.txt
timeout 600 python bench.py --no-cpu-baseline --no-strong --steps 10 > gpurun_out/exp9_bench.json 2> gpurun_out/exp9_bench.err
