# Round-end ncu evidence (one GPU): launch list of bench steps at C4 and --set full of each product
# kernel (incl. the NEXT-4 release kernels via tools/release_probe.py at C2).
set -x
export VLR_GEN_CACHE=/tmp/vlrcache
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none --kernel-name regex:"^(k_|void k_)" \
  --launch-skip 40 --launch-count 30 --csv --log-file gpurun_out/launches_r01_final2.csv \
  python bench.py --steps 4 --warmup 3 --ncu > gpurun_out/ncu_launch_bench.log 2>&1
timeout 2400 ncu --set full --import-source on --clock-control none \
  --kernel-name regex:"k_scan|k_filter_tc|k_exact|k_refine|k_select|k_rank_merge|k_lut8|k_offsets" \
  --launch-skip 40 --launch-count 8 -o gpurun_out/prof_final2 -f \
  python bench.py --steps 4 --warmup 3 --ncu > gpurun_out/ncu_full_bench.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none --kernel-name regex:"k_scan|k_release_merge" \
  --launch-skip 8 --launch-count 3 -o gpurun_out/prof_release -f python tools/release_probe.py > gpurun_out/ncu_rel.log 2>&1
tail -2 gpurun_out/ncu_full_bench.log gpurun_out/ncu_rel.log
