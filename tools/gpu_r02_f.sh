# round 2, call F: exact-theta K2 (candidate band), CTA-parallel item search in the scan, warp item advance,
# K1 adaptive query tile; tests, sanitizers, bench, G=8 model, K1 variants at world 8, workload report C2
set -x
export VLR_GEN_CACHE=/tmp/vlr_gen_cache
python -c "from paper_2504_08930_b200 import build; build.build()" > gpurun_out/build_f.log 2>&1
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu_r02_f.log 2>&1; echo "pytest_rc=$?" >> gpurun_out/pytest_gpu_r02_f.log
timeout 1200 python bench.py > gpurun_out/bench_c4_f.json 2> gpurun_out/bench_c4_f.err
timeout 900 python tools/shard_model.py --config C4 --G 8 --batches 8 > gpurun_out/shard_model_c4_g8_f.json 2> gpurun_out/shard_model_c4_g8_f.err
timeout 600 python tools/k1_bench.py --config C4 --batch 256 --world 8 --rank 3 --variants single,single_tmapB > gpurun_out/k1_bench_w8_f.jsonl 2>&1
for tool in memcheck racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $tool --print-limit 50 python tools/sanitize_run.py > gpurun_out/sanitize_${tool}_f.log 2>&1; echo "rc=$?" >> gpurun_out/sanitize_${tool}_f.log
done
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29543 \
  bench.py --gpus 2 --dry-run-1gpu --exchange staged --config C2 --steps 5 --warmup 3 > gpurun_out/dryrun_c2_n2_staged.json 2> gpurun_out/dryrun_c2_n2_staged.err
tail -3 gpurun_out/pytest_gpu_r02_f.log
