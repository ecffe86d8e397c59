cd $GRAFT_REPO_ROOT
( timeout 900 python -m pytest tests/test_gpu_aggregate.py tests/test_gpu_ddp.py -x -q ) > gpurun_out/t_v.log 2>&1
grep -E "passed|failed" gpurun_out/t_v.log; grep -E "^E " gpurun_out/t_v.log | head -5
for c in mag240m products; do timeout 900 python tools/fused_bench.py --config $c --iters 20 --check 2>&1 | grep -E "avg_us|check"; done
for c in mag240m mag240m papers100m; do
timeout 900 python bench.py --config $c --no-cpu-baseline > gpurun_out/b_v.json 2> gpurun_out/b_v.err
python -c "import json;d=json.load(open('gpurun_out/b_v.json'));print('$c', d['value'],d['ms_per_step'],d['e2e']['value'],d['roofline']['frac'],d['epoch']['seeds_per_s'],d['epoch']['begin_epoch_s'])"
done
