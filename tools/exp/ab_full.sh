# A/B of build variants with the default bench command (e2e + variants legs on), ABAB order
# (run from the repo root under gpurun): tools/exp/ab_full.sh "<label>=<flags>" ...
mkdir -p gpurun_out; : > gpurun_out/ab.txt
for rep in 1 2; do
for v in "$@"; do
  label="${v%%=*}"; flags="${v#*=}"
  GS_NVCC_EXTRA="$flags" python -m paper_2409_06765_b200.build --force > /dev/null || continue
  timeout 600 python bench.py --no-cpu-baseline --no-strong > gpurun_out/ab_$label.json 2>/dev/null
  python -c "
import json,sys
d=json.loads(open('gpurun_out/ab_$label.json').read().strip().splitlines()[-1])
print('$label', d['value'], d['ms_per_step'], {k: v['ms'] for k, v in d['stages'].items()})" >> gpurun_out/ab.txt
done; done
python -m paper_2409_06765_b200.build --force > /dev/null
