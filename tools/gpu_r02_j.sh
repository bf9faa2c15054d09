# round 2, call J (re-entry): HEAD baseline -- full GPU tests, bench C4, G=8 shard model + its launch list
set -x
export VLR_GEN_CACHE=/tmp/vlr_gen_cache
python -c "from paper_2504_08930_b200 import build; build.build()" > gpurun_out/build_j.log 2>&1
timeout 1200 python bench.py > gpurun_out/bench_c4_j.json 2> gpurun_out/bench_c4_j.err
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu_r02_j.log 2>&1; echo "pytest_rc=$?" >> gpurun_out/pytest_gpu_r02_j.log
timeout 900 python tools/shard_model.py --config C4 --G 8 --batches 8 > gpurun_out/shard_model_c4_g8_j.json 2> gpurun_out/shard_model_c4_g8_j.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_shard_g8_j.csv \
  python tools/shard_model.py --config C4 --G 8 --batches 2 > gpurun_out/ncu_shard_j.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --kernel-name regex:"^(k_|void k_)" \
  --launch-skip 40 --launch-count 30 --csv --log-file gpurun_out/launches_c4_j.csv \
  python bench.py --steps 4 --warmup 3 --ncu > gpurun_out/ncu_launch_bench_j.log 2>&1
tail -3 gpurun_out/pytest_gpu_r02_j.log
