# Round-end ncu evidence for profiles/ (run under gpurun, one GPU):
#  1. launch list (gpu__time_duration) of one bench step's kernels at C4
#  2. --set full of one launch of each product kernel at C4, batch 256
set -x
export VLR_GEN_CACHE=/tmp/vlrcache
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none --kernel-name regex:"^(k_|void k_)" \
  --launch-skip 40 --launch-count 30 --csv --log-file gpurun_out/launches_r01_final.csv \
  python bench.py --steps 4 --warmup 3 --ncu > gpurun_out/ncu_launch_bench.log 2>&1
timeout 2400 ncu --set full --import-source on --clock-control none \
  --kernel-name regex:"k_scan|k_filter_tc|k_exact|k_refine|k_select|k_rank_merge|k_lut8|k_offsets" \
  --launch-skip 40 --launch-count 8 -o gpurun_out/prof_final -f \
  python bench.py --steps 4 --warmup 3 --ncu > gpurun_out/ncu_full_bench.log 2>&1
tail -3 gpurun_out/ncu_full_bench.log
