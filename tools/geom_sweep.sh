#!/bin/bash
# development: C2 throughput for several tile geometries (kf,Rf,kb,Rb)
for g in "13,5,12,4" "13,4,12,4" "13,4,12,3" "12,4,12,4" "12,4,11,3" "12,5,12,4" "13,5,12,3"; do
  QF_GEOM_C64=$g python bench.py --batch ${BATCH:-256} --steps 3 --warmup 3 --no-cpu > gpurun_out/geom_$g.json 2>&1
  python -c "
import json; d=json.load(open('gpurun_out/geom_$g.json')); r=d['roofline']
print('$g', round(d['value'],1), d['program'], {k:(round(v['ms'],1), round(v['GBps'] or 0)) for k,v in r['classes'].items()})"
done
