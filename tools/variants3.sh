#!/bin/bash
# development: pipelined (QF_JIT_PIPE=1) kernels x geometry x occupancy (C2, batch ${BATCH:-256})
for spec in "$@"; do
  g=${spec%%/*}; m=${spec##*/}
  QF_JIT_PIPE=1 QF_GEOM_C64=$g QF_JIT_MINB=$m python bench.py --batch ${BATCH:-256} --steps 3 --warmup 3 --no-cpu > "gpurun_out/v3_${g}_$m.json" 2>&1
  python -c "
import json; d=json.load(open('gpurun_out/v3_${g}_$m.json')); r=d['roofline']
print('pipe $g/$m', round(d['value'],1), d['program']['fwd_sweeps'], d['program']['bwd_sweeps'], {k:(round(v['ms'],1), round(v['GBps'] or 0)) for k,v in r['classes'].items() if k!='reduction'})" || tail -2 "gpurun_out/v3_${g}_$m.json"
done
