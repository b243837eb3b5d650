#!/usr/bin/env bash
# One gpurun call: smoke, GPU tests, the default bench line (cfg2) with the CPU
# baseline and the reference arm, the other BASELINE configs, an ncu launch
# list of the default bench and full ncu captures of its dominant kernel and
# of the open-set update.  Outputs: gpurun_out/<tag>_*.
set -u
TAG=${1:-fin}
OUT=gpurun_out
mkdir -p "$OUT"
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,driver_version --format=csv > "$OUT/${TAG}_gpu.txt" 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > "$OUT/${TAG}_smoke.log" 2>&1; echo "smoke rc=$?" >> "$OUT/${TAG}_smoke.log"
[ -z "${NO_TESTS:-}" ] && { timeout 1200 python -m pytest tests -m gpu -x -q > "$OUT/${TAG}_pytest.log" 2>&1; echo "pytest rc=$?" >> "$OUT/${TAG}_pytest.log"; }
timeout 600 python bench.py > "$OUT/${TAG}_bench_cfg2.json" 2> "$OUT/${TAG}_bench_cfg2.err"
timeout 900 python bench.py --impl reference --steps 5 --warmup 3 > "$OUT/${TAG}_bench_ref.json" 2> "$OUT/${TAG}_bench_ref.err"
timeout 600 python bench.py --config 1 --depth --steps 15 --warmup 3 --no-cpu-baseline > "$OUT/${TAG}_bench_cfg1_depth.json" 2> "$OUT/${TAG}_bench_cfg1.err"
timeout 600 python bench.py --config 4 --no-cpu-baseline > "$OUT/${TAG}_bench_cfg4.json" 2> "$OUT/${TAG}_bench_cfg4.err"
timeout 900 python bench.py --config 3 --depth --steps 15 --warmup 3 --no-cpu-baseline > "$OUT/${TAG}_bench_cfg3_depth.json" 2> "$OUT/${TAG}_bench_cfg3.err"
timeout 900 python bench.py --config 5 --depth --steps 10 --warmup 3 --no-cpu-baseline > "$OUT/${TAG}_bench_cfg5_depth.json" 2> "$OUT/${TAG}_bench_cfg5.err"
[ -n "${NO_NCU:-}" ] && exit 0
PCMD="python bench.py --steps 3 --warmup 3 --profile-frames 0 --no-cpu-baseline --no-e2e"
if $PCMD > "$OUT/${TAG}_plain.log" 2>&1; then
  ncu --metrics gpu__time_duration.sum --clock-control none --csv \
      --log-file "$OUT/${TAG}_launches.csv" $PCMD > "$OUT/${TAG}_ncu_launch.log" 2>&1
  ncu --set full --clock-control none --import-source on -k "regex:k_resolve" -s 4 -c 1 \
      -o "$OUT/${TAG}_k_resolve" -f $PCMD > "$OUT/${TAG}_ncu_full.log" 2>&1
fi
ncu --set full --clock-control none --import-source on --kernel-name-base function -k "regex:^k_update_open$" -s 2 -c 1 \
    -o "$OUT/${TAG}_k_update_open_cfg3" -f python tools/mode_diag.py --config 3 --mode auto --frames 3 > "$OUT/${TAG}_ncu_open.log" 2>&1
echo done >> "$OUT/${TAG}_ncu_full.log"
