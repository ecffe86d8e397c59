# dW0 CTA default for P > 128 (96): wgrad/train tests + papers100M A/B vs 111, products unchanged
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r6t
( timeout 900 python -m pytest tests/test_gpu_train.py tests/test_gpu_aggregate.py -m gpu -x -q ) > gpurun_out/r6t/t.log 2>&1
tail -1 gpurun_out/r6t/t.log; grep -E "^E " gpurun_out/r6t/t.log | head
for r in 1 2 3; do
for c in 0 111; do
FG_WGRAD_CTAS=$c timeout 600 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --no-epoch > gpurun_out/r6t/b_${c}_$r.json 2> gpurun_out/r6t/b_${c}_$r.err
python -c "import json;d=json.load(open('gpurun_out/r6t/b_${c}_$r.json'));print('p100m wgrad_ctas=$c', d['value'],d['ms_per_step'],d['e2e']['value'])"
done
done
timeout 600 python bench.py --config products --steps 30 --warmup 5 --no-cpu-baseline --no-epoch > gpurun_out/r6t/b_prod.json 2> gpurun_out/r6t/b_prod.err
python -c "import json;d=json.load(open('gpurun_out/r6t/b_prod.json'));print('products', d['value'],d['ms_per_step'])"
