cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r4c
( timeout 1200 python -m pytest tests/test_gpu_aggregate.py tests/test_gpu_train.py -x -q -m gpu ) > gpurun_out/r4c/t.log 2>&1
tail -1 gpurun_out/r4c/t.log; grep -E "^E |FAIL" gpurun_out/r4c/t.log | head
for v in 1 0; do FG_RELU_BITS=$v timeout 600 python tools/chain_timing.py mag240m 2>&1 | tail -1; done
timeout 900 python bench.py --config mag240m --no-cpu-baseline --no-epoch > gpurun_out/r4c/b_mag.json 2> gpurun_out/r4c/b_mag.err
python -c "import json;d=json.load(open('gpurun_out/r4c/b_mag.json'));print('mag', d['value'],d['ms_per_step'],d['e2e']['value'])"
