# default bench repeatability (papers100M) + kgemm parity test
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r6g
( timeout 600 python -m pytest tests/test_gpu_aggregate.py -m gpu -x -q -k kgemm ) > gpurun_out/r6g/t.log 2>&1; tail -1 gpurun_out/r6g/t.log
for r in 1 2 3; do
timeout 900 python bench.py --no-cpu-baseline --no-epoch > gpurun_out/r6g/b$r.json 2> gpurun_out/r6g/b$r.err
python -c "import json;d=json.load(open('gpurun_out/r6g/b$r.json'));print('p100m', d['value'],d['ms_per_step'],d['e2e']['value'],d['roofline']['avg_launch_us'])"
done
FG_SAGE_KGEMM=0 timeout 900 python bench.py --no-cpu-baseline --no-epoch > gpurun_out/r6g/b_k0.json 2> gpurun_out/r6g/b_k0.err
python -c "import json;d=json.load(open('gpurun_out/r6g/b_k0.json'));print('p100m kgemm0', d['value'],d['ms_per_step'],d['e2e']['value'],d['roofline']['avg_launch_us'])"
