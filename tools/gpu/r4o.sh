cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r4o
for v in 0 1; do
FG_SAGE_KGEMM=$v timeout 600 python tools/chain_timing.py mag240m 2>&1 | tail -1
FG_SAGE_KGEMM=$v timeout 900 python bench.py --config mag240m --no-cpu-baseline --no-epoch > gpurun_out/r4o/b_mag$v.json 2> gpurun_out/r4o/b_mag$v.err
python -c "import json;d=json.load(open('gpurun_out/r4o/b_mag$v.json'));print('mag kgemm=$v', d['value'],d['ms_per_step'],d['e2e']['value'])"
done
FG_SAGE_KGEMM=1 timeout 600 python -m pytest tests/test_gpu_train.py -x -q -m gpu -k "not accuracy" 2>&1 | tail -1
timeout 600 python -m pytest tests/test_gpu_gat.py -x -q -m gpu 2>&1 | tail -1
