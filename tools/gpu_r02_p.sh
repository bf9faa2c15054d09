# round 2, call P: release tail (claims + k_release_rest), PDL only without pipelining, traffic-aware deal
# option -- tests, bench, G=8 model (paper / traffic deal), dry run N=2
set -x
export VLR_GEN_CACHE=/tmp/vlr_gen_cache
python -c "from paper_2504_08930_b200 import build; build.build()" > gpurun_out/build_p.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/pytest_p.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_p.log
timeout 1200 python bench.py > gpurun_out/bench_c4_p.json 2> gpurun_out/bench_c4_p.err
timeout 900 python tools/shard_model.py --config C4 --G 8 --batches 8 --pipe-reserve 0,8,16 > gpurun_out/shard_model_c4_g8_p.json 2> gpurun_out/shard_model_c4_g8_p.err
timeout 900 python tools/shard_model.py --config C4 --G 8 --batches 8 --pipe-reserve 0,8,16 --deal traffic > gpurun_out/shard_model_c4_g8_p_traffic.json 2> gpurun_out/shard_model_c4_g8_p_traffic.err
timeout 600 python tools/scan_trace.py --config C4 --G 1 --release > gpurun_out/scan_trace_rel_p.jsonl 2> gpurun_out/scan_trace_rel_p.err
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29549 \
  bench.py --gpus 2 --dry-run-1gpu --config C2 --steps 10 --warmup 3 --deal traffic > gpurun_out/dryrun_c2_n2_p.json 2> gpurun_out/dryrun_c2_n2_p.err
tail -3 gpurun_out/pytest_p.log
