cd $GRAFT_REPO_ROOT
for c in papers100m mag240m; do
timeout 900 python bench.py --config $c --no-cpu-baseline --steps 5 --warmup 3 > gpurun_out/b_w.json 2> gpurun_out/b_w.err
python -c "import json;d=json.load(open('gpurun_out/b_w.json'));print('$c', d['value'],d['e2e']['value'],d['epoch'])"
done
