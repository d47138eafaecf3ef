# dev-library phase clocks (tools/phase_timing.py); args: extra env assignments
mkdir -p gpurun_out
for e in "$@"; do
  env TTP_DEV_LIBRARY=1 $e timeout 600 python tools/phase_timing.py 2>&1 | head -6 > gpurun_out/phase_$(echo $e | tr '=:' '__').log
  echo "== $e"; cat gpurun_out/phase_$(echo $e | tr '=:' '__').log
done
