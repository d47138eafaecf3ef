mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "decisions or p4 or batch or single or cfg5 or fiber or dev_knob or throughput" > gpurun_out/t_tsqr.log 2>&1; echo "tests rc=$?" >> gpurun_out/t_tsqr.log
tail -5 gpurun_out/t_tsqr.log
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench_tsqr.json 2> gpurun_out/bench_tsqr.err; tail -2 gpurun_out/bench_tsqr.err
python -c "import json;d=json.load(open('gpurun_out/bench_tsqr.json'));print(d['value'],d['e2e']['value'],d['roofline']['avg_launch_ms'],d['parity'])"
TTP_DEV_LIBRARY=1 timeout 600 python tools/phase_timing.py > gpurun_out/phase_tsqr.log 2>&1; head -3 gpurun_out/phase_tsqr.log
TTP_TSQR=0 TTP_DEV_LIBRARY=1 timeout 600 python tools/phase_timing.py > gpurun_out/phase_notsqr.log 2>&1; head -3 gpurun_out/phase_notsqr.log
