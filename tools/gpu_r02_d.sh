# round 2, call D: new generator end-to-end, K1 pre-tiled B, K3a variants, tests, bench with latency leg,
# G=8 per-rank model, scan per-CTA timeline
set -x
export VLR_GEN_CACHE=/tmp/vlr_gen_cache
python -c "from paper_2504_08930_b200 import build; build.build()" > gpurun_out/build_d.log 2>&1
timeout 120 python tools/stall_debug.py > gpurun_out/stall_debug.log 2>&1
timeout 600 python tools/k1_bench.py --config C4 --batch 256 --variants single,single_tmapB,exact_3_2x2,exact_3_4x2,exact_5_2x2,exact_4_4 > gpurun_out/k1_bench_d.jsonl 2>&1
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu_r02_d.log 2>&1; echo "pytest_rc=$?" >> gpurun_out/pytest_gpu_r02_d.log
timeout 1200 python bench.py > gpurun_out/bench_c4_d.json 2> gpurun_out/bench_c4_d.err
for cfg in 3,2 3,6; do VLR_EXACT_CFG=$cfg timeout 600 python bench.py --steps 10 --warmup 3 --no-oracle --lat-batches 0 --sustained-s 0 > gpurun_out/bench_c4_d_exact_${cfg/,/_}.json 2>/dev/null; done
timeout 900 python tools/shard_model.py --config C4 --G 8 --batches 8 > gpurun_out/shard_model_c4_g8_d.json 2> gpurun_out/shard_model_c4_g8_d.err
timeout 900 python tools/scan_trace.py --config C4 --G 1,8 > gpurun_out/scan_trace_c4.jsonl 2> gpurun_out/scan_trace_c4.err
tail -3 gpurun_out/pytest_gpu_r02_d.log
