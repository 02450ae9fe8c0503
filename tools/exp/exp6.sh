mkdir -p gpurun_out
: > gpurun_out/variants.txt
tools/variant_bench.sh "torder="
tools/variant_bench.sh "torder=" -- --config batch3m --views-per-gpu 8
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -4 > gpurun_out/exp6_tests.txt
