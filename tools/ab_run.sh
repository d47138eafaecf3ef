#!/bin/bash
# A/B: GPU parity suite, then bench with the default path and with one
# env switch ($AB_ENV, e.g. TTP_QFORM=zung2r) flipped.
mkdir -p gpurun_out
python -m pytest tests -m gpu -q -x -k "${AB_TESTS:-}" > gpurun_out/gpu_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/gpu_tests.log
env ${AB_ENV:-AB_NONE=1} python bench.py --no-cpu-baseline > gpurun_out/bench_a.json 2> gpurun_out/bench_a.err
python bench.py --no-cpu-baseline > gpurun_out/bench_b.json 2> gpurun_out/bench_b.err
TTP_BOND_PATH=l2:2 python tools/phase_timing.py > gpurun_out/phase.log 2>&1
