# full ncu capture (source-level) of C2's first adjoint sweep at batch 64
python tools/c2_once.py C2 64 > /dev/null
ncu --set full --import-source on --clock-control none -k regex:qf_sweep --launch-skip 31 --launch-count 1 \
    -o gpurun_out/bwd0 python tools/c2_once.py C2 64 > gpurun_out/ncu_bwd0.log 2>&1
echo NCU $?
