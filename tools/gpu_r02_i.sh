# round 2, call I: K2 stage-2 race fix (n_g read vs s_cnt reset) -> sharded tests, G=8 model, bench
set -x
export VLR_GEN_CACHE=/tmp/vlr_gen_cache
python -c "from paper_2504_08930_b200 import build; build.build()" > gpurun_out/build_i.log 2>&1
timeout 900 python -m pytest tests/test_gpu_sharded.py tests/test_gpu_large_k.py tests/test_gpu_multiproc.py -q -x -p no:cacheprovider > gpurun_out/pytest_sharded_i.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_sharded_i.log
timeout 900 python tools/shard_model.py --config C4 --G 8 --batches 8 > gpurun_out/shard_model_c4_g8_i.json 2> gpurun_out/shard_model_c4_g8_i.err
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu_r02_i.log 2>&1; echo "pytest_rc=$?" >> gpurun_out/pytest_gpu_r02_i.log
timeout 1200 python bench.py > gpurun_out/bench_c4_i.json 2> gpurun_out/bench_c4_i.err
tail -3 gpurun_out/pytest_sharded_i.log; tail -3 gpurun_out/pytest_gpu_r02_i.log; cat gpurun_out/shard_model_c4_g8_i.json | head -c 1500
