timeout 1200 ncu --set full --import-source on --clock-control none --kernel-name regex:"k_rank_merge|k_select|k_exact|k_refine|k_lut8|k_filter_tc|k_offsets|k_qprep" --launch-skip 0 --launch-count 18 -o gpurun_out/prof_small -f python tools/stages.py --N 8000000 --batches 1,256 > gpurun_out/ncu_small.log 2>&1
tail -3 gpurun_out/ncu_small.log
