cd $GRAFT_REPO_ROOT
( timeout 1800 python -m pytest tests/test_gpu_aggregate.py tests/test_gpu_fullscale.py tests/test_gpu_train.py -x -q ) > gpurun_out/t_q.log 2>&1
grep -E "passed|failed" gpurun_out/t_q.log; grep -E "^E " gpurun_out/t_q.log | head -8
for e in 1 0; do FG_SQ_LANE=$e timeout 900 python tools/fused_bench.py --config papers100m --iters 20 --check 2>&1 | grep -E "avg_us|check"; done
FG_SQ_LANE=1 timeout 900 python tools/fused_bench.py --config arxiv --iters 20 --check 2>&1 | grep -E "avg_us|check"
FG_SQ_LANE=0 timeout 900 python tools/fused_bench.py --config arxiv --iters 20 --check 2>&1 | grep -E "avg_us|check"
timeout 900 python bench.py --no-cpu-baseline --no-epoch > gpurun_out/b_q.json 2> gpurun_out/b_q.err
python -c "import json;d=json.load(open('gpurun_out/b_q.json'));print('papers100m', d['value'],d['ms_per_step'],d['e2e']['value'],d['roofline']['frac'],d['roofline']['avg_launch_us'])"
