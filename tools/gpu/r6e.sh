# MAG: chunked dW0 GEMM (16 slices, default on the GEMM path) vs one cuBLAS GEMM
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r6e
for v in 0 auto 0 auto; do
FG_SAGE_KGEMM=$v timeout 900 python bench.py --config mag240m --steps 20 --warmup 5 --no-cpu-baseline --no-epoch > gpurun_out/r6e/b_mag_$v.json 2> gpurun_out/r6e/b_mag_$v.err
python -c "import json;d=json.load(open('gpurun_out/r6e/b_mag_$v.json'));print('mag kgemm=$v', d['value'],d['ms_per_step'],d['e2e']['value'])"
done
( timeout 900 python -m pytest tests/test_gpu_train.py -m gpu -x -q ) > gpurun_out/r6e/t.log 2>&1; tail -1 gpurun_out/r6e/t.log
