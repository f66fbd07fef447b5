# 4 concurrent builds of the C2 program against one empty JIT cache, then the
# single-process baseline against another empty cache.
export QF_JIT_CACHE=/tmp/qf_share_$$
rm -rf $QF_JIT_CACHE
t0=$(date +%s%N)
for i in 1 2 3 4; do python tools/jit_share_probe.py C2 & done; wait
echo "4 concurrent: $(( ($(date +%s%N) - t0) / 1000000 )) ms"
export QF_JIT_CACHE=/tmp/qf_single_$$
rm -rf $QF_JIT_CACHE
python tools/jit_share_probe.py C2
ls /tmp/qf_share_$$ | grep -c lock
