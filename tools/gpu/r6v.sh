# end-of-session check: full gpu suite + smoke + default bench line (with cpu_baseline) + GAT line
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r6v
( time timeout 2400 python -m pytest tests -m gpu -q ) > gpurun_out/r6v/t_gpu_all.log 2>&1
tail -2 gpurun_out/r6v/t_gpu_all.log
( timeout 600 python -c "import __graft_entry__ as g; g.smoke()" ) > gpurun_out/r6v/smoke.log 2>&1; tail -1 gpurun_out/r6v/smoke.log
timeout 900 python bench.py > gpurun_out/r6v/bench_papers100m.json 2> gpurun_out/r6v/bench_papers100m.err
timeout 900 python bench.py --config mag240m --no-cpu-baseline > gpurun_out/r6v/bench_mag240m.json 2> gpurun_out/r6v/bench_mag240m.err
timeout 900 python bench.py --config products-gat --no-cpu-baseline > gpurun_out/r6v/bench_products-gat.json 2> gpurun_out/r6v/bench_products-gat.err
for f in gpurun_out/r6v/bench_*.json; do echo $f; python -c "import json,sys;d=json.load(open('$f'));print(d.get('value'),d.get('ms_per_step'),d.get('e2e',{}).get('value'),(d.get('roofline') or {}).get('frac'),(d.get('epoch') or {}).get('seeds_per_s'))"; done
