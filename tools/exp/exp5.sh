mkdir -p gpurun_out
: > gpurun_out/variants.txt
tools/variant_bench.sh "base=" "order=-DGS_TILE_ORDER=1"
tools/variant_bench.sh "base=" "order=-DGS_TILE_ORDER=1" -- --config batch3m --views-per-gpu 8
tools/variant_bench.sh "base=" "order=-DGS_TILE_ORDER=1" -- --config large6m --views-per-gpu 4
