# round 2 end evidence on the final build: GPU tests, smoke, bench (headline line), reference arm, ncu launch
# list and one --set full capture of the step's kernels (summarised into profiles/r02/ by the caller)
set -x
export VLR_GEN_CACHE=/tmp/vlr_gen_cache
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/final_build.log 2>&1
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/final_pytest_gpu.log 2>&1; echo "pytest_rc=$?" >> gpurun_out/final_pytest_gpu.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final_smoke.log 2>&1; echo "smoke_rc=$?" >> gpurun_out/final_smoke.log
timeout 1200 python bench.py > gpurun_out/final_bench.json 2> gpurun_out/final_bench.err
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/final_reference.json 2> gpurun_out/final_reference.err
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --kernel-name regex:"^(k_|void k_)" \
  --launch-skip 40 --launch-count 30 --csv --log-file gpurun_out/final_launches.csv \
  python bench.py --steps 4 --warmup 3 --ncu > gpurun_out/final_ncu_launch.log 2>&1
timeout 2400 ncu --set full --import-source on --clock-control none \
  --kernel-name regex:"k_scan|k_filter_tc|k_exact|k_refine|k_select|k_rank_merge|k_lut8|k_offsets|k_qprep" \
  --launch-skip 40 --launch-count 9 -o gpurun_out/final_prof -f \
  python bench.py --steps 4 --warmup 3 --ncu > gpurun_out/final_ncu_full.log 2>&1
python tools/ncu_summary.py gpurun_out/final_prof.ncu-rep gpurun_out/final_ncu_full.json "round-2 final build, C4 batch 256" > /dev/null 2>&1
tail -3 gpurun_out/final_pytest_gpu.log; tail -2 gpurun_out/final_smoke.log; head -c 300 gpurun_out/final_bench.json
