#!/bin/bash
# Round-2 evidence on one B200 (run under gpurun): bench line (cfg3 headline +
# cfg4 apply), the reference arm, the cfg2 line, the launch list of the bench
# command, full ncu captures of the layer histogram (cfg3, one tree: layers
# 1-5), the refresh / list advance and the apply kernel, and the free-running
# divergence report.  .ncu-rep files stay in /tmp on the box (gpurun_out/ is
# capped at 64 MiB); only their text summaries come back.
mkdir -p gpurun_out
python bench.py > gpurun_out/r02_bench.json 2> gpurun_out/r02_bench.err
python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/r02_bench_ref.json 2>> gpurun_out/r02_bench.err
python bench.py --config cfg2 --no-apply --no-cpu > gpurun_out/r02_bench_cfg2.json 2>> gpurun_out/r02_bench.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 4000 --csv --log-file /tmp/r02_launches_bench.csv \
    python bench.py --steps 1 --warmup 3 --no-apply --no-e2e --no-cpu > gpurun_out/r02_ncu_bench.log 2>&1
python tools/ncu_summary.py launches /tmp/r02_launches_bench.csv gpurun_out/r02_launches_bench_cfg3.txt
ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file /tmp/r02_launches_8.csv \
    python tools/prof_fit.py --config cfg3 --trees 8 --reps 1 > gpurun_out/r02_ncu_fit8.log 2>&1
python tools/ncu_summary.py launches /tmp/r02_launches_8.csv gpurun_out/r02_launches_fit_cfg3_8trees.txt
ncu --set full --import-source on --clock-control none -k regex:k_hist_list -c 5 -o /tmp/r02_hist_full \
    python tools/prof_fit.py --config cfg3 --trees 1 --reps 1 --host-masks > gpurun_out/r02_ncu_hist.log 2>&1
python tools/ncu_summary.py full /tmp/r02_hist_full.ncu-rep gpurun_out/r02_ncu_full_hist_cfg3.txt
python tools/ncu_summary.py traffic /tmp/r02_hist_full.ncu-rep gpurun_out/r02_hist_traffic_cfg3.json
ncu --set full --import-source on --clock-control none -k regex:"k_update_refresh|k_advance_list" -c 14 -o /tmp/r02_tree_full \
    python tools/prof_fit.py --config cfg3 --trees 2 --reps 1 --host-masks > gpurun_out/r02_ncu_tree.log 2>&1
python tools/ncu_summary.py full /tmp/r02_tree_full.ncu-rep gpurun_out/r02_ncu_full_refresh_advance_cfg3.txt
ncu --set full --import-source on --clock-control none -k regex:k_apply -c 1 -o /tmp/r02_apply_full \
    python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu --apply-rows 10000000 --config cfg1 > gpurun_out/r02_ncu_apply.log 2>&1
python tools/ncu_summary.py full /tmp/r02_apply_full.ncu-rep gpurun_out/r02_ncu_full_apply.txt
python tools/divergence.py > gpurun_out/r02_divergence.txt 2>&1
ls -la gpurun_out | tail -30
