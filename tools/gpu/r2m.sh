# round-2: adaptive compaction / seed sort; GAT step profile
cd $GRAFT_REPO_ROOT
( timeout 1200 python -m pytest tests/test_gpu_sampler.py -x -q ) > gpurun_out/t_samp.log 2>&1
grep -E "passed|failed" gpurun_out/t_samp.log; grep -E "Error|assert" gpurun_out/t_samp.log | head -5
timeout 600 python tools/chain_timing.py products > gpurun_out/chain_prod.txt 2>&1; tail -1 gpurun_out/chain_prod.txt
timeout 600 python bench.py --config products --steps 20 --warmup 5 --no-cpu-baseline --no-epoch > gpurun_out/b_lp.json 2> gpurun_out/b_lp.err
python -c "import json;d=json.load(open('gpurun_out/b_lp.json'));print('products', d['value'],d['ms_per_step'],d['roofline']['avg_launch_us'],d['e2e']['value'])"
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-epoch > gpurun_out/b_l.json 2> gpurun_out/b_l.err
python -c "import json;d=json.load(open('gpurun_out/b_l.json'));print('papers100m', d['value'],d['ms_per_step'],d['roofline']['avg_launch_us'],d['e2e']['value'])"
timeout 900 ncu --nvtx --nvtx-include "step/" --metrics gpu__time_duration.sum \
    --clock-control none --csv --log-file gpurun_out/launches_gat.csv \
    python tools/profile_step.py --config products-gat --steps 2 > gpurun_out/prof_gat.log 2>&1
tail -2 gpurun_out/prof_gat.log
timeout 600 python bench.py --config products-gat --steps 10 --warmup 3 --no-cpu-baseline --no-epoch > gpurun_out/b_gat.json 2> gpurun_out/b_gat.err
python -c "import json;d=json.load(open('gpurun_out/b_gat.json'));print('gat', d['value'],d['ms_per_step'])"
