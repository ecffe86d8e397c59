cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r5f
( timeout 1200 python -m pytest tests/test_gpu_gat.py -x -q -m gpu ) > gpurun_out/r5f/t.log 2>&1
tail -1 gpurun_out/r5f/t.log; grep -E "^E |Error" gpurun_out/r5f/t.log | head -20
for v in 1; do
FG_GAT_EXPLICIT=$v timeout 900 python bench.py --config products-gat --steps 10 --warmup 3 --no-cpu-baseline --no-epoch > gpurun_out/r5f/b_gat$v.json 2> gpurun_out/r5f/b_gat$v.err
python -c "import json;d=json.load(open('gpurun_out/r5f/b_gat$v.json'));print('gat explicit=$v', d['value'],d['ms_per_step'],d['e2e']['value'])"
tail -2 gpurun_out/r5f/b_gat$v.err
done
timeout 900 ncu --nvtx --nvtx-include "step/" --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/r5f/launches_products-gat_step.csv python tools/profile_step.py --config products-gat --steps 2 > gpurun_out/r5f/prof_gat.log 2>&1
tail -1 gpurun_out/r5f/prof_gat.log
