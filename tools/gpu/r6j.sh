# staged host-seed H2D: parity test + e2e A/B (papers100m default, products-gat)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r6j
( timeout 900 python -m pytest tests/test_gpu_train.py -m gpu -x -q -k "host_seeds or pipelined" ) > gpurun_out/r6j/t.log 2>&1
tail -1 gpurun_out/r6j/t.log; grep -E "^E " gpurun_out/r6j/t.log | head
for r in 1 2 3; do
timeout 900 python bench.py --no-cpu-baseline --no-epoch > gpurun_out/r6j/b$r.json 2> gpurun_out/r6j/b$r.err
python -c "import json;d=json.load(open('gpurun_out/r6j/b$r.json'));print('p100m', d['value'],d['ms_per_step'],d['e2e']['value'])"
done
timeout 900 python bench.py --config products-gat --no-cpu-baseline --no-epoch > gpurun_out/r6j/bg.json 2> gpurun_out/r6j/bg.err
python -c "import json;d=json.load(open('gpurun_out/r6j/bg.json'));print('gat', d['value'],d['ms_per_step'],d['e2e']['value'])"
