# round 2, call B: K1 CTA-pair kernel correctness + variant timing, tests, shard model, bench
set -x
python -c "from paper_2504_08930_b200 import build; build.build()" > gpurun_out/build_b.log 2>&1
timeout 300 python tools/k1_bench.py --config C4 --batch 256 > gpurun_out/k1_bench_c4_b256.jsonl 2>&1
timeout 300 python tools/k1_bench.py --config C4 --batch 256 --world 8 --rank 3 --variants pair,single,pair_qt64,pair_qt128 > gpurun_out/k1_bench_c4_b256_w8.jsonl 2>&1
timeout 300 python tools/k1_bench.py --config C4 --batch 32 --variants pair,single > gpurun_out/k1_bench_c4_b32.jsonl 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_gpu_r02_b.log 2>&1; echo "pytest_rc=$?" >> gpurun_out/pytest_gpu_r02_b.log
timeout 900 python tools/shard_model.py --config C4 --G 8 --batches 8 > gpurun_out/shard_model_c4_g8_b.json 2> gpurun_out/shard_model_c4_g8_b.err
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_c4_b.json 2> gpurun_out/bench_c4_b.err
tail -3 gpurun_out/pytest_gpu_r02_b.log
