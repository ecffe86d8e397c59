# round-2 re-entry check: GAT suite + smoke + default and GAT bench lines after the last GAT commits
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r6a
( time timeout 1200 python -m pytest tests/test_gpu_gat.py tests/test_gpu_aggregate.py -m gpu -x -q ) > gpurun_out/r6a/t.log 2>&1
tail -3 gpurun_out/r6a/t.log
( timeout 600 python -c "import __graft_entry__ as g; g.smoke()" ) > gpurun_out/r6a/smoke.log 2>&1; tail -1 gpurun_out/r6a/smoke.log
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/r6a/b_def.json 2> gpurun_out/r6a/b_def.err
timeout 900 python bench.py --config products-gat --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/r6a/b_gat.json 2> gpurun_out/r6a/b_gat.err
for f in gpurun_out/r6a/b_*.json; do echo $f; python -c "import json,sys;d=json.load(open('$f'));print(d.get('value'),d.get('ms_per_step'),d.get('e2e',{}).get('value'),(d.get('roofline') or {}).get('frac'),(d.get('epoch') or {}).get('seeds_per_s'))"; done
