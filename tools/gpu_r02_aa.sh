# round 2, call AA: plain-scan A/B, product vs VLR_SCAN_SMEMQ=1 variant (events around K6)
set -x
export VLR_GEN_CACHE=/tmp/vlr_gen_cache
python -c "from paper_2504_08930_b200 import build; build.build()" > gpurun_out/build_aa.log 2>&1
timeout 600 python tools/variant_parity.py smemq > gpurun_out/variant_parity_smemq_aa.log 2>&1
for lib in product smemq product smemq product smemq; do
  timeout 600 python tools/scan_ab.py $lib >> gpurun_out/scan_ab_aa.jsonl 2>> gpurun_out/scan_ab_aa.err
done
cat gpurun_out/scan_ab_aa.jsonl; tail -2 gpurun_out/variant_parity_smemq_aa.log
