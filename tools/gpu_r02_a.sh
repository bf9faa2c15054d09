# round 2, call A: GPU tests (incl. the sharded coarse stage, NCCL timeouts, 2-process gloo),
# the N=2 dry run of bench.py on one GPU, the G=8 per-rank model at C4, and a C4 bench line.
set -x
python -c "from paper_2504_08930_b200 import build; build.build()" > gpurun_out/build_a.log 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_gpu_r02_a.log 2>&1; echo "pytest_rc=$?" >> gpurun_out/pytest_gpu_r02_a.log
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 \
  bench.py --gpus 2 --dry-run-1gpu --config C2 --steps 5 --warmup 3 > gpurun_out/dryrun_c2_n2.json 2> gpurun_out/dryrun_c2_n2.err
timeout 900 python tools/shard_model.py --config C4 --G 8 --batches 8 > gpurun_out/shard_model_c4_g8.json 2> gpurun_out/shard_model_c4_g8.err
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_c4_a.json 2> gpurun_out/bench_c4_a.err
tail -3 gpurun_out/pytest_gpu_r02_a.log
