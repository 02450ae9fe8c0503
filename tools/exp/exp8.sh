mkdir -p gpurun_out
: > gpurun_out/variants.txt
tools/variant_bench.sh "base=" "half=-DGS_K7_HALF=1"
tools/variant_bench.sh "base=" "half=-DGS_K7_HALF=1" -- --config batch3m --views-per-gpu 8
GS_NVCC_EXTRA=-DGS_K7_HALF=1 python -m paper_2409_06765_b200.build --force > /dev/null
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "backward or tile_order or absgrad or depth or nd_features or graph" 2>&1 | tail -3 > gpurun_out/exp8_tests.txt
python -m paper_2409_06765_b200.build --force > /dev/null
