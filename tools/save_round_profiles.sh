#!/bin/bash
# Copy the outputs of tools/r2_final.sh (gpurun_out/) into profiles/ (round-2 names).
set -e
grep '^{' gpurun_out/v_bench.log | tail -1 > profiles/r2_bench_c2.json
grep '^{' gpurun_out/v_bench_ref.log | tail -1 > profiles/r2_bench_c2_reference_arm.json
cp gpurun_out/prof_launches.csv profiles/r2_ncu_launches_c2.csv
python tools/ncu_summary.py gpurun_out/prof_bwd0.ncu-rep > profiles/r2_ncu_full_c2_b1024_bwd0.txt 2>&1
ncu -i gpurun_out/prof_bwd0.ncu-rep --page source --csv --print-source sass > /tmp/bwd0_src.csv 2>/dev/null || true
python tools/sass_mix.py /tmp/bwd0_src.csv 16 >> profiles/r2_ncu_full_c2_b1024_bwd0.txt 2>&1 || true
python tools/ncu_summary.py gpurun_out/prof_hpsi.ncu-rep > profiles/r2_ncu_full_c2_b1024_hpsi.txt 2>&1
for c in C1 C3 C4 C5; do grep '^{' gpurun_out/f_bench_$c.json | tail -1 > profiles/r2_bench_$c.json; done
tail -1 gpurun_out/f_mipt.json > profiles/r2_bench_mipt_tableIV.json
cp gpurun_out/f_noise.jsonl profiles/r2_bench_noise_trajectories.jsonl
{
  echo "# round-2 end verification of HEAD (tools/r2_final.sh) on one B200"
  tail -2 gpurun_out/v_smoke.log; tail -2 gpurun_out/v_pytest.log; tail -2 gpurun_out/v_dropin.log
  echo "torchrun --nproc-per-node 1 bench.py: $(tail -1 gpurun_out/f_torchrun.log)"
  python - <<'PY'
import json
d = json.load(open('profiles/r2_bench_c2.json')); r = d['roofline']
print('C2 bench:', round(d['value'], 1), 'evals/s; e2e', round(d['e2e']['value'], 1), '; c128', round(d['c128']['value'], 1),
      '; binding roofline', r['bound'], round(r['frac'], 3), '(hbm', round(r['hbm']['frac'], 3), '); clocks', d['clocks'])
for c in ['C1', 'C3', 'C4', 'C5']:
    d = json.load(open('profiles/r2_bench_%s.json' % c))
    print(c + ':', round(d['value'], 3), 'evals/s; e2e', round(d['e2e']['value'], 3))
d = json.load(open('profiles/r2_bench_mipt_tableIV.json'))
print('MIPT Table IV:', round(d['s_per_traj'], 5), 's/traj')
PY
} > profiles/r2_verify.txt
cat profiles/r2_verify.txt
