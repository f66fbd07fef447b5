# Dump the generated sweep sources of C2 and capture the first adjoint sweep
# (launch 31 of qf_sweep... selected by -k/--launch-skip) at batch 64 with ncu --set full.
mkdir -p gpurun_out/jitdump
QF_JIT_DUMP=gpurun_out/jitdump QF_JIT_CACHE=/tmp/qf_dump_$$ python tools/c2_once.py C2 64 > gpurun_out/dump_once.log 2>&1; echo ONCE $?
ncu --set full --import-source on --clock-control none -k regex:qf_sweep --launch-skip 9 --launch-count 2 \
    -o gpurun_out/bwd0b python tools/c2_once.py C2 64 > gpurun_out/ncu_bwd0b.log 2>&1
echo NCU $?
