#!/usr/bin/env bash
# One gpurun call: GPU parity tests, the default bench line, the bench with
# the CPU baseline, an ncu launch list and one `ncu --set full` capture of the
# top kernel.  Usage (from the build container):
#   gpurun --timeout 2400 -- 'bash tools/gpu_check.sh <tag> [kernel-regex]'
# Outputs land in gpurun_out/<tag>_*.
set -u
TAG=${1:-run}
KRE=${2:-k_resolve}
OUT=gpurun_out
mkdir -p "$OUT"
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,driver_version --format=csv > "$OUT/${TAG}_gpu.txt" 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > "$OUT/${TAG}_smoke.log" 2>&1
echo "smoke rc=$?" >> "$OUT/${TAG}_smoke.log"
[ -z "${NO_TESTS:-}" ] && timeout 1500 python -m pytest tests -m gpu -x -q > "$OUT/${TAG}_pytest.log" 2>&1
echo "pytest rc=$?" >> "$OUT/${TAG}_pytest.log"
timeout 600 python bench.py > "$OUT/${TAG}_bench.json" 2> "$OUT/${TAG}_bench.err"
echo "bench rc=$?" >> "$OUT/${TAG}_bench.err"
timeout 300 python tools/host_overhead.py > "$OUT/${TAG}_host.txt" 2>&1
timeout 300 python tools/host_overhead.py --mode segments >> "$OUT/${TAG}_host.txt" 2>&1
SVX_TRACE_HOST=1 timeout 300 python tools/host_overhead.py --frames 12 > "$OUT/${TAG}_host_trace.txt" 2>&1
[ -n "${WITH_REF:-}" ] && timeout 600 python bench.py --impl reference --steps 5 --warmup 3 > "$OUT/${TAG}_bench_ref.json" 2> "$OUT/${TAG}_bench_ref.err"
echo "ref rc=$?" >> "$OUT/${TAG}_bench_ref.err" 2>/dev/null
PCMD="python bench.py --steps 3 --warmup 3 --profile-frames 0 --no-cpu-baseline --no-e2e"
if [ -z "${NO_NCU:-}" ] && $PCMD > "$OUT/${TAG}_plain.log" 2>&1; then
  ncu --metrics gpu__time_duration.sum --clock-control none --csv \
      --log-file "$OUT/${TAG}_launches.csv" $PCMD > "$OUT/${TAG}_ncu_launch.log" 2>&1
  ncu --set full --clock-control none --import-source on -k "regex:${KRE}" -s 4 -c 2 \
      -o "$OUT/${TAG}_prof" -f $PCMD > "$OUT/${TAG}_ncu_full.log" 2>&1
  echo "ncu done" >> "$OUT/${TAG}_ncu_full.log"
fi
