# A/B of one dev knob on the GPU box: interleaved bench runs of the dev library
# with $AB_ENV (A) and without (B), then the dev phase clocks of both.
# Usage: AB_ENV="TTP_START_FILTER=0" AB_TESTS="dev_knob or decisions" bash tools/gpu/ab_env.sh
mkdir -p gpurun_out
if [ -n "${AB_TESTS:-}" ]; then
  timeout 1200 python -m pytest tests -m gpu -x -q -k "$AB_TESTS" > gpurun_out/t_ab.log 2>&1; echo "tests rc=$?" >> gpurun_out/t_ab.log
  tail -4 gpurun_out/t_ab.log
fi
for rep in 1 2; do
  for arm in A B; do
    if [ $arm = A ]; then e="$AB_ENV"; else e="AB_NONE=1"; fi
    env TTP_DEV_LIBRARY=1 $e timeout 600 python bench.py --no-cpu-baseline --steps ${AB_STEPS:-5} > gpurun_out/bench_$arm$rep.json 2> gpurun_out/bench_$arm$rep.err
    python -c "import json;d=json.load(open('gpurun_out/bench_$arm$rep.json'));print('$arm$rep', d['value'],d['e2e']['value'],d['roofline']['avg_launch_ms'],d['parity']['max_rel'], d['parity']['ok'])" 2>&1 | tail -1
  done
done
env TTP_DEV_LIBRARY=1 $AB_ENV PT_CASES=4:148 timeout 600 python tools/phase_timing.py 2>&1 | head -4 > gpurun_out/phase_A.log
env TTP_DEV_LIBRARY=1 PT_CASES=4:148 timeout 600 python tools/phase_timing.py 2>&1 | head -4 > gpurun_out/phase_B.log
echo "== A ($AB_ENV)"; cat gpurun_out/phase_A.log; echo "== B"; cat gpurun_out/phase_B.log
