# VQ lane: 768-thread variant on MAG; products step with the 512-thread default (W=4) vs 1024; parity tests
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r6i
( timeout 900 python -m pytest tests/test_gpu_aggregate.py tests/test_gpu_fullscale.py tests/test_gpu_train.py -m gpu -x -q ) > gpurun_out/r6i/t.log 2>&1
tail -1 gpurun_out/r6i/t.log; grep -E "^E " gpurun_out/r6i/t.log | head
for nt in 1024 768 1024 768; do
FG_VQ_LANE_NT=$nt timeout 600 python tools/fused_bench.py --config mag240m --iters 40 > gpurun_out/r6i/fb_mag_$nt.txt 2>&1
echo "mag $nt: $(tail -1 gpurun_out/r6i/fb_mag_$nt.txt | python -c 'import json,sys;d=json.loads(sys.stdin.read());print(d["avg_us"],d["min_us"],d["frac"])')"
done
for nt in 1024 0 1024 0; do
FG_VQ_LANE_NT=$nt timeout 900 python bench.py --config products --no-cpu-baseline --no-epoch > gpurun_out/r6i/b_prod_$nt.json 2> gpurun_out/r6i/b_prod_$nt.err
python -c "import json;d=json.load(open('gpurun_out/r6i/b_prod_$nt.json'));print('products nt=$nt', d['value'],d['ms_per_step'],d['e2e']['value'],d['roofline']['avg_launch_us'])"
done
