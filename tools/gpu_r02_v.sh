# round 2, call V: per-warp item cache in the scan's loads (VLR_SCAN_ICACHE=1 variant) -- bitwise check vs the
# product library, scan traces at G = 1 and 8 (A/B interleaved)
set -x
export VLR_GEN_CACHE=/tmp/vlr_gen_cache
python -c "from paper_2504_08930_b200 import build; build.build()" > gpurun_out/build_v.log 2>&1
timeout 600 python tools/variant_parity.py ic > gpurun_out/variant_parity_ic_v.log 2>&1; echo "rc=$?" >> gpurun_out/variant_parity_ic_v.log
for lib in scantrace scantrace_ic scantrace scantrace_ic; do
  timeout 600 python tools/scan_trace.py --config C4 --G 1,8 --lib $lib >> gpurun_out/scan_trace_ic_v.jsonl 2>> gpurun_out/scan_trace_ic_v.err
done
cat gpurun_out/variant_parity_ic_v.log
