#!/bin/bash
# A/B with the switch ON in run a (tests run with it too).
mkdir -p gpurun_out
env ${AB_ENV} python -m pytest tests -m gpu -q -x > gpurun_out/gpu_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/gpu_tests.log
env ${AB_ENV} python bench.py --no-cpu-baseline --no-e2e > gpurun_out/bench_a.json 2> gpurun_out/bench_a.err
python bench.py --no-cpu-baseline --no-e2e > gpurun_out/bench_b.json 2> gpurun_out/bench_b.err
env ${AB_ENV} TTP_BOND_PATH=l2:2 python tools/phase_timing.py > gpurun_out/phase.log 2>&1
