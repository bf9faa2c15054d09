# round 2, call Z: confirmation on the last build (release-scan register fix): GPU tests, smoke, bench,
# ncu launch list
set -x
export VLR_GEN_CACHE=/tmp/vlr_gen_cache
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/zz_build.log 2>&1
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/zz_pytest_gpu.log 2>&1; echo "pytest_rc=$?" >> gpurun_out/zz_pytest_gpu.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/zz_smoke.log 2>&1; echo "smoke_rc=$?" >> gpurun_out/zz_smoke.log
timeout 1200 python bench.py > gpurun_out/zz_bench.json 2> gpurun_out/zz_bench.err
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --kernel-name regex:"^(k_|void k_)" \
  --launch-skip 40 --launch-count 30 --csv --log-file gpurun_out/zz_launches.csv \
  python bench.py --steps 4 --warmup 3 --ncu > gpurun_out/zz_ncu_launch.log 2>&1
tail -3 gpurun_out/zz_pytest_gpu.log; tail -2 gpurun_out/zz_smoke.log; head -c 300 gpurun_out/zz_bench.json
