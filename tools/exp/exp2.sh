set -x
mkdir -p gpurun_out
GS_NVCC_EXTRA=-DGS_K7_STATS python -m paper_2409_06765_b200.build --force > /dev/null && timeout 300 python tools/k7_stats.py > gpurun_out/exp2_k7stats.txt 2>&1
: > gpurun_out/variants.txt
tools/variant_bench.sh "base=" "match=-DGS_SCATTER_MATCH=1"
tools/variant_bench.sh "base=" "match=-DGS_SCATTER_MATCH=1" -- --config batch3m --views-per-gpu 8
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "isect or config2 or packed_parity" 2>&1 | tail -3 > gpurun_out/exp2_tests.txt
