# Round-end verification of HEAD on one B200: smoke, GPU tests, C++ drop-in checks, bench (ours + reference arm)
set -x
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/v_smoke.log 2>&1; echo smoke=$? >> gpurun_out/v_smoke.log
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/v_pytest.log 2>&1; echo pytest=$? >> gpurun_out/v_pytest.log
timeout 300 ./cpp/test_dropin > gpurun_out/v_dropin.log 2>&1; echo dropin=$? >> gpurun_out/v_dropin.log
timeout 600 python bench.py > gpurun_out/v_bench.log 2>&1; echo bench=$? >> gpurun_out/v_bench.log
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/v_bench_ref.log 2>&1; echo bench_ref=$? >> gpurun_out/v_bench_ref.log
