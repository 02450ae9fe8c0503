mkdir -p gpurun_out
: > gpurun_out/variants.txt
tools/variant_bench.sh "L8=" "L1=-DGS_PBWD_MAXL=1" "L4=-DGS_PBWD_MAXL=4" -- --config batch3m --views-per-gpu 8
tools/variant_bench.sh "L8=" "L1=-DGS_PBWD_MAXL=1" -- --config large6m --views-per-gpu 4
tools/variant_bench.sh "L8=" -- --config aa_packed1m --views-per-gpu 4
tools/variant_bench.sh "L8="
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -4 > gpurun_out/exp4_tests.txt
