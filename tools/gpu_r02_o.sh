# round 2, call O: release scan with alternating segment order + out-of-order merger (Z = 1); PDL chain;
# gmeta reverted -- full tests, bench, PDL A/B, G=8 model, release trace
set -x
export VLR_GEN_CACHE=/tmp/vlr_gen_cache
python -c "from paper_2504_08930_b200 import build; build.build()" > gpurun_out/build_o.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/pytest_o.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_o.log
timeout 1200 python bench.py --lat-batches 0 --sustained-s 0 > gpurun_out/bench_c4_o.json 2> gpurun_out/bench_c4_o.err
VLR_PDL=0 timeout 1200 python bench.py --lat-batches 0 --sustained-s 0 --no-oracle --e2e-steps 4 > gpurun_out/bench_c4_o_nopdl.json 2> gpurun_out/bench_c4_o_nopdl.err
timeout 1200 python bench.py --lat-batches 0 --sustained-s 0 --no-oracle --e2e-steps 4 > gpurun_out/bench_c4_o_pdl2.json 2> gpurun_out/bench_c4_o_pdl2.err
timeout 900 python tools/shard_model.py --config C4 --G 8 --batches 8 > gpurun_out/shard_model_c4_g8_o.json 2> gpurun_out/shard_model_c4_g8_o.err
VLR_PDL=0 timeout 900 python tools/shard_model.py --config C4 --G 8 --batches 8 --pipe-reserve 0,16 > gpurun_out/shard_model_c4_g8_o_nopdl.json 2> gpurun_out/shard_model_c4_g8_o_nopdl.err
timeout 600 python tools/scan_trace.py --config C4 --G 1 --release > gpurun_out/scan_trace_rel_o.jsonl 2> gpurun_out/scan_trace_rel_o.err
tail -3 gpurun_out/pytest_o.log
