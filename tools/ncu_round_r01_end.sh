# Round-end ncu evidence for the final build (one GPU): launch list of bench steps at C4
# (cold-cache, serialised per-launch times: compare shares, not absolutes) and --set full
# of the product kernels. The LUT kernel runs on its side stream; ncu serialises it.
set -x
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --kernel-name regex:"^(k_|void k_)" \
  --launch-skip 40 --launch-count 30 --csv --log-file gpurun_out/launches_r01_end.csv \
  python bench.py --steps 4 --warmup 3 --ncu > gpurun_out/ncu_launch_bench.log 2>&1
timeout 1800 ncu --set full --import-source on --clock-control none \
  --kernel-name regex:"k_scan|k_filter_tc|k_exact|k_refine|k_select|k_rank_merge|k_lut8|k_offsets" \
  --launch-skip 40 --launch-count 8 -o gpurun_out/prof_r01_end -f \
  python bench.py --steps 4 --warmup 3 --ncu > gpurun_out/ncu_full_bench.log 2>&1
tail -2 gpurun_out/ncu_launch_bench.log gpurun_out/ncu_full_bench.log
