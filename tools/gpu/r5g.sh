cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r5g
for v in 1 0 1 0; do
FG_GAT_OVERLAP=$v timeout 900 python bench.py --config products-gat --steps 30 --warmup 3 --no-cpu-baseline --no-epoch > gpurun_out/r5g/b_gat$v.json 2> gpurun_out/r5g/b_gat$v.err
python -c "import json;d=json.load(open('gpurun_out/r5g/b_gat$v.json'));print('gat overlap=$v', d['value'],d['ms_per_step'],d['e2e']['value'])"
done
