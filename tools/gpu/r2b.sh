# round-2: gpu suite, full-scale parity, fused-kernel A/B (v4 sliced vs v5 lane-per-part)
cd $GRAFT_REPO_ROOT
( time timeout 1800 python -m pytest tests -m gpu -x -q --deselect tests/test_gpu_world.py --deselect tests/test_gpu_fullscale.py -k "not config_a" ) > gpurun_out/t_gpu.log 2>&1
( time timeout 1500 python -m pytest tests/test_gpu_fullscale.py -x -q -s ) > gpurun_out/t_full.log 2>&1
( time timeout 1200 python -m pytest tests/test_gpu_train.py -x -q -s -k config_a ) > gpurun_out/t_acc.log 2>&1
for c in products mag240m; do for l in 0 1; do
  FG_VQ_LANE=$l timeout 600 python tools/fused_bench.py --config $c --iters 20 --check >> gpurun_out/fused_ab.jsonl 2>> gpurun_out/fused_ab.err
done; done
tail -3 gpurun_out/t_gpu.log gpurun_out/t_full.log gpurun_out/t_acc.log; cat gpurun_out/fused_ab.jsonl
