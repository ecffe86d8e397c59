# round-2: wgrad v2 correctness + timing; lane-f16 default for MAG; papers100m bench + chains
cd $GRAFT_REPO_ROOT
( timeout 900 python -m pytest tests/test_gpu_aggregate.py -x -q ) > gpurun_out/t_agg.log 2>&1
grep -E "passed|failed" gpurun_out/t_agg.log
for v in 0 1; do for P in 112 144; do
  FG_WGRAD_V2=$v timeout 300 python tools/wgrad_probe.py $P >> gpurun_out/wgrad.txt 2>&1
done; done
cat gpurun_out/wgrad.txt | grep median
( timeout 1200 python -m pytest tests/test_gpu_train.py -x -q ) > gpurun_out/t_train.log 2>&1
grep -E "passed|failed" gpurun_out/t_train.log
timeout 600 python tools/chain_timing.py papers100m > gpurun_out/chain_p100m.txt 2>&1; tail -1 gpurun_out/chain_p100m.txt
timeout 600 python tools/chain_timing.py products > gpurun_out/chain_prod.txt 2>&1; tail -1 gpurun_out/chain_prod.txt
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-epoch > gpurun_out/b_k.json 2> gpurun_out/b_k.err
python -c "import json;d=json.load(open('gpurun_out/b_k.json'));print('papers100m', d['value'],d['ms_per_step'],d['roofline']['avg_launch_us'],d['e2e']['value'])"
timeout 600 python tools/fused_bench.py --config mag240m --iters 20 --check > gpurun_out/mag_def.json 2>&1; grep -E "avg_us|check" gpurun_out/mag_def.json
