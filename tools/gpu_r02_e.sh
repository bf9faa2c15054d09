# round 2, call E: tests incl. the peer exchange (2 processes, 1 GPU), dry-run N=2 (p2p and staged),
# candidate-band stats on the new data, per-kernel launch list of the G=8 per-rank model, sanitizers
set -x
export VLR_GEN_CACHE=/tmp/vlr_gen_cache
python -c "from paper_2504_08930_b200 import build; build.build()" > gpurun_out/build_e.log 2>&1
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu_r02_e.log 2>&1; echo "pytest_rc=$?" >> gpurun_out/pytest_gpu_r02_e.log
timeout 600 python tools/band_stats.py --config C4 > gpurun_out/band_stats_c4.json 2>&1
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29541 \
  bench.py --gpus 2 --dry-run-1gpu --exchange p2p --config C2 --steps 5 --warmup 3 > gpurun_out/dryrun_c2_n2_p2p.json 2> gpurun_out/dryrun_c2_n2_p2p.err
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29542 \
  bench.py --gpus 2 --dry-run-1gpu --exchange staged --config C2 --steps 5 --warmup 3 > gpurun_out/dryrun_c2_n2_staged.json 2> gpurun_out/dryrun_c2_n2_staged.err
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --kernel-name regex:"^(k_|void k_|vlr)" --csv --log-file gpurun_out/launches_shard_g8_c4.csv python tools/shard_model.py --config C4 --G 8 --batches 1 --warmup 1 > gpurun_out/ncu_shard_c4.log 2>&1
for tool in memcheck racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $tool --print-limit 50 python tools/sanitize_run.py > gpurun_out/sanitize_${tool}.log 2>&1; echo "rc=$?" >> gpurun_out/sanitize_${tool}.log
done
timeout 900 env VLR_FILTER_CLUSTER=2 compute-sanitizer --tool racecheck --print-limit 50 python tools/sanitize_run.py > gpurun_out/sanitize_racecheck_cl2.log 2>&1; echo "rc=$?" >> gpurun_out/sanitize_racecheck_cl2.log
timeout 900 env VLR_FILTER_PAIR=1 compute-sanitizer --tool racecheck --print-limit 50 python tools/sanitize_run.py > gpurun_out/sanitize_racecheck_pair.log 2>&1; echo "rc=$?" >> gpurun_out/sanitize_racecheck_pair.log
tail -3 gpurun_out/pytest_gpu_r02_e.log
