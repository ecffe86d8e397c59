cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r4m
( timeout 1500 python -m pytest tests/test_gpu_gat.py tests/test_gpu_sampler.py tests/test_gpu_aggregate.py -x -q -m gpu ) > gpurun_out/r4m/t.log 2>&1
tail -1 gpurun_out/r4m/t.log; grep -E "^E |Error" gpurun_out/r4m/t.log | head -20
timeout 900 python bench.py --config products-gat --steps 10 --warmup 3 --no-cpu-baseline --no-epoch > gpurun_out/r4m/b_gat.json 2> gpurun_out/r4m/b_gat.err
python -c "import json;d=json.load(open('gpurun_out/r4m/b_gat.json'));print('gat', d['value'],d['ms_per_step'],d['e2e']['value'])"
timeout 900 ncu --nvtx --nvtx-include "step/" --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/r4m/launches_products-gat_step.csv python tools/profile_step.py --config products-gat --steps 2 > gpurun_out/r4m/prof_gat.log 2>&1
tail -1 gpurun_out/r4m/prof_gat.log
