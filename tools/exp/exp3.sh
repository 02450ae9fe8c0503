mkdir -p gpurun_out
: > gpurun_out/variants.txt
tools/variant_bench.sh "d3pass="
tools/variant_bench.sh "d3pass=" -- --config batch3m --views-per-gpu 8
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -4 > gpurun_out/exp3_tests.txt
