cd $GRAFT_REPO_ROOT
( timeout 1800 python -m pytest tests/test_gpu_train.py tests/test_gpu_aggregate.py -x -q ) > gpurun_out/t_g.log 2>&1
grep -E "passed|failed" gpurun_out/t_g.log; grep -E "^E " gpurun_out/t_g.log | head -5
for c in products products-gcn papers100m; do
timeout 900 python bench.py --config $c --no-cpu-baseline --no-epoch > gpurun_out/b_g.json 2> gpurun_out/b_g.err
python -c "import json;d=json.load(open('gpurun_out/b_g.json'));print('$c', d['value'],d['ms_per_step'],d['e2e']['value'])"
done
timeout 600 python tools/chain_timing.py papers100m > gpurun_out/chain_p.txt 2>&1; tail -1 gpurun_out/chain_p.txt
