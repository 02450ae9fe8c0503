mkdir -p gpurun_out
python -m paper_2409_06765_b200.build > /dev/null
: > gpurun_out/variants.txt
for r in 1 2; do
GS_EXP_LISTLEN=1 tools/variant_bench.sh "listlen="
tools/variant_bench.sh "walk="
done
GS_EXP_LISTLEN=1 tools/variant_bench.sh "listlen=" -- --config batch3m --views-per-gpu 8
tools/variant_bench.sh "walk=" -- --config batch3m --views-per-gpu 8
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "tile_order or backward_parity" 2>&1 | tail -3 > gpurun_out/exp7_tests.txt
