#!/bin/bash
# round 2 verification after the n>=29 fix: all GPU tests, bench (c128 leg), compute-sanitizer memcheck/racecheck
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q --durations=15 > gpurun_out/v7_pytest.log 2>&1; echo pytest=$? >> gpurun_out/v7_pytest.log
timeout 900 python bench.py > gpurun_out/v7_bench.json 2> gpurun_out/v7_bench.err; echo bench=$? >> gpurun_out/v7_bench.err
timeout 900 compute-sanitizer --tool memcheck --print-limit 50 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/v7_memcheck_smoke.log 2>&1; echo rc=$? >> gpurun_out/v7_memcheck_smoke.log
timeout 1200 compute-sanitizer --tool memcheck --print-limit 50 python -m pytest tests/test_gpu_api.py -x -q -k "basic_gates or complex64_mode or sparse_energy or device_entry" > gpurun_out/v7_memcheck_api.log 2>&1; echo rc=$? >> gpurun_out/v7_memcheck_api.log
timeout 900 compute-sanitizer --tool racecheck --print-limit 50 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/v7_racecheck_smoke.log 2>&1; echo rc=$? >> gpurun_out/v7_racecheck_smoke.log
