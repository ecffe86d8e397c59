cd $GRAFT_REPO_ROOT
( timeout 1800 python -m pytest tests/test_gpu_aggregate.py tests/test_gpu_refsuite.py tests/test_gpu_fullscale.py -x -q ) > gpurun_out/t_p.log 2>&1
grep -E "passed|failed" gpurun_out/t_p.log; grep -E "^E " gpurun_out/t_p.log | head -8
for pe in 1 0; do FG_VQ_PAIR=$pe timeout 900 python tools/fused_bench.py --config mag240m --iters 20 --check 2>&1 | grep -E "avg_us|check"; done
