#!/bin/bash
# development: C2 throughput for adjoint geometries / register budgets
run() {  # tag, env...
  local tag=$1; shift
  env "$@" python bench.py --batch ${BATCH:-256} --steps 3 --warmup 3 --no-cpu > gpurun_out/g_$tag.json 2>&1
  python -c "
import json; d=json.load(open('gpurun_out/g_$tag.json')); r=d['roofline']
print('$tag', round(d['value'],1), d['program'], {k:(round(v['ms'],1), round(v['GBps'] or 0)) for k,v in r['classes'].items()})" 2>&1 | tail -1
}
run base QF_GEOM_C64=13,5,12,4
run b12r5m1 QF_GEOM_C64=13,5,12,5 QF_JIT_MINB_BWD=1
run b13r5m1 QF_GEOM_C64=13,5,13,5 QF_JIT_MINB_BWD=1
run b13r4 QF_GEOM_C64=13,5,13,4
run b11r4 QF_GEOM_C64=13,5,11,4
run b12r3m3 QF_GEOM_C64=13,5,12,3 QF_JIT_MINB_BWD=3
