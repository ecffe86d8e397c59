cd $GRAFT_REPO_ROOT
( timeout 1500 python -m pytest tests/test_gpu_aggregate.py tests/test_gpu_fullscale.py -x -q ) > gpurun_out/t_x.log 2>&1
grep -E "passed|failed" gpurun_out/t_x.log; grep -E "^E " gpurun_out/t_x.log | head -5
for c in mag240m products; do timeout 900 python tools/fused_bench.py --config $c --iters 20 --check 2>&1 | grep -E "avg_us|check"; done
