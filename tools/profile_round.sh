#!/bin/bash
# Round evidence on one B200 (run under gpurun): bench line, ncu launch list of
# the bench command, full ncu captures of the histogram, the parse chain and
# the apply kernel, per-layer histogram times per path (cfg2, cfg3).
mkdir -p gpurun_out
python bench.py > gpurun_out/bench_full.json 2> gpurun_out/bench_full.err
python bench.py --config cfg3 --steps 2 --warmup 1 --no-apply --no-cpu > gpurun_out/bench_cfg3.json 2> gpurun_out/bench_cfg3.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 800 --csv --log-file gpurun_out/launches_bench.csv \
    python bench.py --steps 1 --warmup 3 --no-apply --no-e2e --no-cpu > gpurun_out/ncu_bench.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:k_layer_hist -s 3 -c 3 -o gpurun_out/hist_full \
    python tools/prof_fit.py --trees 4 --reps 1 --host-masks > gpurun_out/ncu_hist.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:k_seg_chain -s 4 -c 1 -o gpurun_out/chain_full \
    python tools/time_masks.py --trees 8 --reps 1 > gpurun_out/ncu_chain.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:k_apply -c 1 -o gpurun_out/apply_full \
    python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu --apply-rows 10000000 > gpurun_out/ncu_apply.log 2>&1
PF_DEPTH=3 bash tools/hist_paths.sh > gpurun_out/hist_paths_cfg2.txt 2>&1
PF_DEPTH=5 PF_ARGS="--config cfg3 --trees 4 --reps 1 --host-masks" bash tools/hist_paths.sh > gpurun_out/hist_paths_cfg3.txt 2>&1
ls -la gpurun_out
