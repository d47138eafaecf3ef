#!/bin/bash
# A/B on the GPU box: the release library against the -DTTP_DEV library with
# one knob flipped ($AB_ENV, e.g. "TTP_SWAP_FILTER=0" or "TTP_LAZY=3"), each
# through bench.py, then the dev library's phase clocks.  The release library
# reads no environment; only the dev build honours TTP_* knobs.
mkdir -p gpurun_out
python -m pytest tests -m gpu -q -x -k "${AB_TESTS:-}" > gpurun_out/gpu_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/gpu_tests.log
env TTP_DEV_LIBRARY=1 ${AB_ENV:-AB_NONE=1} python bench.py --no-cpu-baseline > gpurun_out/bench_a.json 2> gpurun_out/bench_a.err
python bench.py --no-cpu-baseline > gpurun_out/bench_b.json 2> gpurun_out/bench_b.err
python tools/phase_timing.py > gpurun_out/phase.log 2>&1
