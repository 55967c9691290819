#!/bin/bash
# Round profiling artefacts (run under gpurun): bench JSON, ncu launch list,
# one full ncu capture of the dominant kernel.  Output in gpurun_out/.
set -u
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 600 python bench.py --steps 3 --warmup 3 > gpurun_out/bench_full.json 2> gpurun_out/bench_full.err
echo "bench rc=$?"
# launch list: plain run first (must exit 0), then the same command under ncu
CMD="python bench.py --steps 1 --warmup 3 --no-cpu-baseline"
timeout 300 $CMD > gpurun_out/plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -s 30000 -c 4000 --csv \
    --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launch.log 2>&1
echo "launch list rc=$?"
# dominant kernel, full set, fine grid (255^3 red-black sweep with fused prolongation)
KB="python tools/kernel_bench.py --n 256 --reps 1 --only vcycle_jor-rb_V11"
timeout 120 $KB > /dev/null 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_zrb -s 4 -c 2 \
    -o gpurun_out/zrb255_full $KB > gpurun_out/ncu_full.log 2>&1
echo "full capture rc=$?"
