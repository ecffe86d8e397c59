# round-2: presorted seeds (no seed-sort kernel), batched k-means++ kernel, SQ register-kernel A/B
cd $GRAFT_REPO_ROOT
( timeout 2400 python -m pytest tests/test_gpu_sampler.py tests/test_gpu_train.py tests/test_gpu_ddp.py tests/test_gpu_codecs.py tests/test_gpu_fullscale.py tests/test_gpu_gat.py -x -q ) > gpurun_out/t_r.log 2>&1
grep -E "passed|failed" gpurun_out/t_r.log; grep -E "^E |Error" gpurun_out/t_r.log | head -8
timeout 900 python bench.py --no-cpu-baseline --no-epoch > gpurun_out/b_r.json 2> gpurun_out/b_r.err
python -c "import json;d=json.load(open('gpurun_out/b_r.json'));print('papers100m', d['value'],d['ms_per_step'],d['e2e']['value'])"
FG_SQ_BULK=0 timeout 900 python tools/fused_bench.py --config papers100m --iters 20 --check 2>&1 | grep -E "avg_us|check"
timeout 900 python bench.py --config products --no-cpu-baseline --no-epoch > gpurun_out/b_rp.json 2> gpurun_out/b_rp.err
python -c "import json;d=json.load(open('gpurun_out/b_rp.json'));print('products', d['value'],d['ms_per_step'],d['e2e']['value'])"
timeout 900 python bench.py --config mag240m --no-cpu-baseline --no-epoch > gpurun_out/b_rm.json 2> gpurun_out/b_rm.err
python -c "import json;d=json.load(open('gpurun_out/b_rm.json'));print('mag240m', d['value'],d['ms_per_step'],d['e2e']['value'])"; grep "vq codec" gpurun_out/b_rm.err
