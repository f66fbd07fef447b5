#!/bin/bash
# development: alternate A/B runs of bench.py under two env settings: ab.sh "ENV_A" "ENV_B" [reps]
A=$1; B=$2; N=${3:-2}
for i in $(seq 1 $N); do
  for tag in A B; do
    if [ $tag = A ]; then E=$A; else E=$B; fi
    env $E python bench.py --steps 3 --warmup 3 --no-cpu ${BENCH_ARGS} > gpurun_out/ab_$tag.json 2>&1
    python -c "
import json; d=json.load(open('gpurun_out/ab_$tag.json')); r=d['roofline']
print('$tag', '$E', round(d['value'],1), round(d['e2e']['value'],1), d['clocks']['sm_mhz'], d['clocks']['reasons'], {k:round(v['ms'],1) for k,v in r['classes'].items()})" 2>&1 | tail -1
  done
done
