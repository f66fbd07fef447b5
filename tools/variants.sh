#!/bin/bash
# development: compare JIT variants on C2 (batch ${BATCH:-256})
run() { tag=$1; shift; env "$@" python bench.py --batch ${BATCH:-256} --steps 3 --warmup 3 --no-cpu > gpurun_out/var_$tag.json 2>&1;
  python -c "
import json; d=json.load(open('gpurun_out/var_$tag.json')); r=d['roofline']
print('$tag', round(d['value'],1), {k:(round(v['ms'],1), round(v['GBps'] or 0)) for k,v in r['classes'].items()}, round(d['program']['jit']['seconds'],1))" || tail -3 gpurun_out/var_$tag.json; }
for v in "$@"; do run $v $(echo $v | tr '+' ' '); done
