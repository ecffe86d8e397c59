cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r5e
for c in 64 32 16; do
FG_KGEMM_CHUNKS=$c timeout 900 python bench.py --config products-gat --steps 20 --warmup 3 --no-cpu-baseline --no-epoch > gpurun_out/r5e/b_gat$c.json 2> gpurun_out/r5e/b_gat$c.err
python -c "import json;d=json.load(open('gpurun_out/r5e/b_gat$c.json'));print('gat chunks=$c', d['value'],d['ms_per_step'],d['e2e']['value'])"
done
