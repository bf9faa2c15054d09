# K3a (S stages, W warps) sweep at C4: parity subset + stage time per configuration (VLR_EXACT_CFG=S,W)
export VLR_GEN_CACHE=/tmp/vlrc
for cfg in 4,4 2,4 3,4 2,8 2,2 4,2 4,4; do
  VLR_EXACT_CFG=$cfg timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -k "golden_tiny_on_gpu or c1_parity or adversarial or overflow or m_variants" > gpurun_out/k3a_pytest_${cfg/,/_}.log 2>&1
  echo "cfg $cfg pytest rc=$? $(tail -1 gpurun_out/k3a_pytest_${cfg/,/_}.log)" >> gpurun_out/k3a_sweep.txt
  VLR_EXACT_CFG=$cfg timeout 400 python bench.py --ncu --steps 30 --warmup 5 > gpurun_out/k3a_bench_${cfg/,/_}.json 2>/dev/null
  python -c "
import json;d=json.loads(open('gpurun_out/k3a_bench_${cfg/,/_}.json').read().strip().splitlines()[-1])
print('cfg $cfg', 'refine_ms', round(d['stage_ms']['refine'],4), 'ms_per_step', round(d['ms_per_step'],4), 'scan', round(d['roofline']['ms_per_launch'],4))" >> gpurun_out/k3a_sweep.txt 2>&1
done
cat gpurun_out/k3a_sweep.txt
