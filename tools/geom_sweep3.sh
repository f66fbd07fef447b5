#!/bin/bash
# development: larger tiles at one 512-thread CTA per SM (same warps/SM as 2 x 256)
run() {
  local tag=$1; shift
  env "$@" python bench.py --batch 256 --steps 3 --warmup 3 --no-cpu > gpurun_out/g_$tag.json 2>&1
  python -c "
import json; d=json.load(open('gpurun_out/g_$tag.json')); r=d['roofline']
print('$tag', round(d['value'],1), d['program']['fwd_sweeps'], d['program']['bwd_sweeps'], {k:round(v['ms'],1) for k,v in r['classes'].items()})" 2>&1 | tail -1
}
run base X=1
run b13r4m1 QF_GEOM_C64=13,5,13,4 QF_JIT_MINB_BWD=1
run f14r5m1 QF_GEOM_C64=14,5,12,4 QF_JIT_MINB_FWD=1
run f14b13m1 QF_GEOM_C64=14,5,13,4 QF_JIT_MINB=1
