# quick A/B on the GPU box: targeted GPU tests, bench, dev phase clocks
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "${AB_TESTS:-decisions or p4 or batch or single or cfg5 or fiber or dev_knob or throughput}" > gpurun_out/t_ab.log 2>&1; echo "tests rc=$?" >> gpurun_out/t_ab.log
tail -4 gpurun_out/t_ab.log
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench_ab.json 2> gpurun_out/bench_ab.err; tail -2 gpurun_out/bench_ab.err
python -c "import json;d=json.load(open('gpurun_out/bench_ab.json'));print('BENCH', d['value'],d['e2e']['value'],d['roofline']['avg_launch_ms'],d['parity']['max_rel'], d['parity']['ok'])"
TTP_DEV_LIBRARY=1 timeout 600 python tools/phase_timing.py 2>&1 | head -6 > gpurun_out/phase_ab.log; cat gpurun_out/phase_ab.log
