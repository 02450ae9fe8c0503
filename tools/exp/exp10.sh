mkdir -p gpurun_out
: > gpurun_out/variants.txt
tools/variant_bench.sh "colors="
tools/variant_bench.sh "colors=" -- --config batch3m --views-per-gpu 8
tools/variant_bench.sh "colors=" -- --config aa_packed1m --views-per-gpu 4
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -4 > gpurun_out/exp10_tests.txt
