# full ncu capture of C2's H|psi> + energy kernel at batch 256 (second evaluation)
python tools/c2_once.py C2 256 > /dev/null
ncu --set full --import-source on --clock-control none -k regex:hpsi --launch-skip 1 --launch-count 1 \
    -o gpurun_out/hpsi python tools/c2_once.py C2 256 > gpurun_out/ncu_hpsi.log 2>&1
echo NCU $?
