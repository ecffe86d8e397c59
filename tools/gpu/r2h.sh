# round-2: v6 (pipelined producer) VQ + SQ fused kernels, infwd v2 -- correctness + A/B
cd $GRAFT_REPO_ROOT
( timeout 900 python -m pytest tests/test_gpu_aggregate.py -x -q ) > gpurun_out/t_agg.log 2>&1
tail -3 gpurun_out/t_agg.log
for c in papers100m products mag240m; do
  for env in "FG_VQ_V6=0 FG_SQ_V6=0" "FG_VQ_V6=1 FG_SQ_V6=1"; do
    env $env timeout 600 python tools/fused_bench.py --config $c --iters 20 --check >> gpurun_out/v6b_ab.jsonl 2>> gpurun_out/v6b_ab.err
    echo "$c $env" >> gpurun_out/v6b_ab.jsonl
  done
done
cat gpurun_out/v6b_ab.jsonl; grep check gpurun_out/v6b_ab.err
for env in "FG_INFWD_V2=0 FG_SQ_V6=0" "FG_INFWD_V2=1 FG_SQ_V6=0" "FG_INFWD_V2=1 FG_SQ_V6=1"; do
  env $env timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-epoch > gpurun_out/b_ab.json 2> gpurun_out/b_ab.err
  echo "$env $(python -c "import json;d=json.load(open('gpurun_out/b_ab.json'));print(d['value'],d['ms_per_step'],d['roofline']['avg_launch_us'],d['e2e']['value'])")" >> gpurun_out/bench_ab.txt
done
cat gpurun_out/bench_ab.txt
( timeout 1200 python -m pytest tests/test_gpu_train.py -x -q ) > gpurun_out/t_train.log 2>&1
tail -3 gpurun_out/t_train.log
