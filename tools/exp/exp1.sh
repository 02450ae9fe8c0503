set -x
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "isect or config2 or packed_parity" 2>&1 | tail -3 > gpurun_out/exp1_tests.txt
GS_NVCC_EXTRA=-DGS_K7_STATS python -m paper_2409_06765_b200.build --force > /dev/null && timeout 300 python tools/k7_stats.py > gpurun_out/exp1_k7stats.txt 2>&1
: > gpurun_out/variants.txt
tools/variant_bench.sh "base=" "vis4=-DGS_VIS_ITEMS=4" "histat=-DGS_HIST_ATOMIC=1" "vis8=-DGS_VIS_ITEMS=8"
tools/variant_bench.sh "base=" "vis4=-DGS_VIS_ITEMS=4" "histat=-DGS_HIST_ATOMIC=1" -- --config batch3m --views-per-gpu 8
