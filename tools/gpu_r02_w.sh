# round 2, call W: N = 2 plumbing at the headline config (C4), two processes on one GPU, peer exchange +
# pipelining, paper deal and traffic-aware deal (not a multi-GPU rate: the processes time-slice one GPU)
set -x
export VLR_GEN_CACHE=/tmp/vlr_gen_cache
python -c "from paper_2504_08930_b200 import build; build.build()" > gpurun_out/build_w.log 2>&1
timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29551 \
  bench.py --gpus 2 --dry-run-1gpu --config C4 --steps 10 --warmup 3 > gpurun_out/dryrun_c4_n2_w.json 2> gpurun_out/dryrun_c4_n2_w.err
timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29553 \
  bench.py --gpus 2 --dry-run-1gpu --config C4 --steps 10 --warmup 3 --deal traffic > gpurun_out/dryrun_c4_n2_traffic_w.json 2> gpurun_out/dryrun_c4_n2_traffic_w.err
tail -c 600 gpurun_out/dryrun_c4_n2_w.json
