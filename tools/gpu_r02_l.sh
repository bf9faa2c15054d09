# round 2, call L: K3b rank-merge (sharded stage 3), K1 query tile at world 8, pipelined G=8 model, tests
set -x
export VLR_GEN_CACHE=/tmp/vlr_gen_cache
python -c "from paper_2504_08930_b200 import build; build.build()" > gpurun_out/build_l.log 2>&1
timeout 900 python -m pytest tests/test_gpu_sharded.py tests/test_gpu_pipeline.py tests/test_gpu_multiproc.py tests/test_gpu_parity.py -q -x -p no:cacheprovider > gpurun_out/pytest_l.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_l.log
timeout 900 python tools/k1_bench.py --config C4 --batch 256 --world 8 --rank 3 --variants single,single_nn32,single_nn64,single_nn128,single_nn256 > gpurun_out/k1_bench_w8_l.jsonl 2>&1
timeout 600 python tools/k1_bench.py --config C4 --batch 256 --world 1 --variants single,single_nn128 > gpurun_out/k1_bench_w1_l.jsonl 2>&1
timeout 900 python tools/shard_model.py --config C4 --G 8 --batches 8 > gpurun_out/shard_model_c4_g8_l.json 2> gpurun_out/shard_model_c4_g8_l.err
tail -3 gpurun_out/pytest_l.log; cat gpurun_out/k1_bench_w8_l.jsonl
timeout 600 python -m pytest tests/test_gpu_release.py -q -x -p no:cacheprovider > gpurun_out/pytest_rel_l.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_rel_l.log
timeout 600 python tools/scan_trace.py --config C4 --G 1 --release > gpurun_out/scan_trace_rel_l.jsonl 2> gpurun_out/scan_trace_rel_l.err
timeout 1200 python bench.py --lat-batches 0 --sustained-s 0 --no-oracle > gpurun_out/bench_c4_l.json 2> gpurun_out/bench_c4_l.err
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29547 \
  bench.py --gpus 2 --dry-run-1gpu --config C2 --steps 10 --warmup 3 > gpurun_out/dryrun_c2_n2_l.json 2> gpurun_out/dryrun_c2_n2_l.err
tail -3 gpurun_out/pytest_rel_l.log; cat gpurun_out/scan_trace_rel_l.jsonl | cut -c1-400
