# round-2: sampler (seed radix sort, 8-item compaction tiles) parity + timing
cd $GRAFT_REPO_ROOT
( timeout 1200 python -m pytest tests/test_gpu_sampler.py tests/test_gpu_fullscale.py -x -q ) > gpurun_out/t_samp.log 2>&1
grep -E "passed|failed" gpurun_out/t_samp.log; grep -E "Error|assert" gpurun_out/t_samp.log | head -5
timeout 600 python tools/chain_timing.py papers100m > gpurun_out/chain_p100m.txt 2>&1; tail -1 gpurun_out/chain_p100m.txt
timeout 600 python tools/chain_timing.py products > gpurun_out/chain_prod.txt 2>&1; tail -1 gpurun_out/chain_prod.txt
for v in 0 1; do
FG_INFWD_V2=$v timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-epoch > gpurun_out/b_l.json 2> gpurun_out/b_l.err
python -c "import json;d=json.load(open('gpurun_out/b_l.json'));print('papers100m infwd_v2=$v', d['value'],d['ms_per_step'],d['roofline']['avg_launch_us'],d['e2e']['value'])"
done
timeout 600 python bench.py --config products --steps 20 --warmup 5 --no-cpu-baseline --no-epoch > gpurun_out/b_lp.json 2> gpurun_out/b_lp.err
python -c "import json;d=json.load(open('gpurun_out/b_lp.json'));print('products', d['value'],d['ms_per_step'],d['roofline']['avg_launch_us'],d['e2e']['value'])"
