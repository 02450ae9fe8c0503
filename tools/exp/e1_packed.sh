mkdir -p gpurun_out
for c in "batch3m 8" "large6m 4" "garden1m 1"; do set -- $c
  for pk in "" "--packed"; do
    echo "== $1 $pk" >> gpurun_out/e1.txt
    timeout 600 python bench.py --config $1 --views-per-gpu $2 $pk --no-cpu-baseline --no-e2e --no-strong --no-variants --steps 10 2>>gpurun_out/e1.err | python -c "
import json,sys;d=json.loads(sys.stdin.read());print(d['value'],d['ms_per_step'],{k:v['ms'] for k,v in d['stages'].items()})" >> gpurun_out/e1.txt 2>&1
  done
done
