#!/bin/bash
# Round profiling artefacts (run under gpurun): bench JSON (default + single-
# stream A/B), ncu launch list of one PFASST block, full ncu captures of the
# top kernels at 255^3.  Output in gpurun_out/; summarise with
# tools/summarize_profiles.py <round>.
set -u
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/bench_full.json 2> gpurun_out/bench_full.err
echo "bench rc=$?"
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-other-configs --no-streams \
    > gpurun_out/bench_nostreams.json 2> gpurun_out/bench_nostreams.err
echo "bench (single stream) rc=$?"
# launch list: plain run first (must exit 0), then the same command under ncu
CMD="python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-other-configs"
timeout 300 $CMD > gpurun_out/plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -s 30000 -c 4000 --csv \
    --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launch.log 2>&1
echo "launch list rc=$?"
# top kernels, full set, on the fine grid (one launch each)
KB="python tools/kernel_bench.py --n 256 --reps 1 --only vcycle_jor-rb_V11,interp_cubic_add"
timeout 120 $KB > /dev/null 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on \
    -k regex:"k_zrb3|k_rfw|k_cubic5|k_mid|k_z1" -c 10 -o gpurun_out/top255_full $KB \
    > gpurun_out/ncu_full.log 2>&1
echo "full capture rc=$?"
# the other fine-level kernels (one launch each): an SDC sweep, the residual, the FAS machinery
KO="python tools/kernel_bench.py --n 256 --reps 1 --only sweep_M8_jorrb_V11,residual_max_M8,restrict_state,compute_fas,coarse_correction"
timeout 200 $KO > /dev/null 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on \
    -k regex:"k_z1|k_cubic5|k_prolong3_cell|k_chain|k_resmax|k_delta_chain" -c 160 -o gpurun_out/other255_full $KO \
    > gpurun_out/ncu_other.log 2>&1
echo "other kernels capture rc=$?"
