# round 2, call X: NEXT-4 device timeline (merger vs k_release_rest), C4
set -x
export VLR_GEN_CACHE=/tmp/vlr_gen_cache
python -c "from paper_2504_08930_b200 import build; build.build()" > gpurun_out/build_x.log 2>&1
timeout 900 python tools/release_timeline.py --config C4 > gpurun_out/release_timeline_x.json 2> gpurun_out/release_timeline_x.err
tail -3 gpurun_out/release_timeline_x.err; head -c 3000 gpurun_out/release_timeline_x.json
