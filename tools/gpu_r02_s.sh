# round 2, call S: alternating segment order for every scan (VLR_SCAN_ALT) -- A/B traces and benches, tests
set -x
export VLR_GEN_CACHE=/tmp/vlr_gen_cache
python -c "from paper_2504_08930_b200 import build; build.build()" > gpurun_out/build_s.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_sharded.py tests/test_gpu_large_k.py tests/test_gpu_release.py -q -x -p no:cacheprovider > gpurun_out/pytest_s.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_s.log
timeout 600 python tools/scan_trace.py --config C4 --G 1,8 > gpurun_out/scan_trace_alt1_s.jsonl 2> gpurun_out/scan_trace_alt1_s.err
VLR_SCAN_ALT=0 timeout 600 python tools/scan_trace.py --config C4 --G 1,8 > gpurun_out/scan_trace_alt0_s.jsonl 2> gpurun_out/scan_trace_alt0_s.err
timeout 600 python tools/scan_trace.py --config C4 --G 1 > gpurun_out/scan_trace_alt1b_s.jsonl 2> gpurun_out/scan_trace_alt1b_s.err
for alt in 0 1 0 1; do
  VLR_SCAN_ALT=$alt timeout 900 python bench.py --no-oracle --steps 30 --lat-batches 0 --sustained-s 0 --e2e-steps 4 \
    >> gpurun_out/bench_alt_s.jsonl 2>> gpurun_out/bench_alt_s.err
done
tail -2 gpurun_out/pytest_s.log
