# round-2: 256-bit output stores in the fused kernels; lane kernel with fp16 table
cd $GRAFT_REPO_ROOT
( timeout 900 python -m pytest tests/test_gpu_aggregate.py -x -q ) > gpurun_out/t_agg.log 2>&1
( FG_VQ_LANE=2 timeout 900 python -m pytest tests/test_gpu_aggregate.py -x -q -k vq ) >> gpurun_out/t_agg.log 2>&1
grep -E "passed|failed" gpurun_out/t_agg.log
for c in papers100m products mag240m; do
  for env in "FG_VQ_LANE=0" "FG_VQ_LANE=2"; do
    env $env timeout 600 python tools/fused_bench.py --config $c --iters 20 --probe 0,3 --check >> gpurun_out/st256.jsonl 2>> gpurun_out/st256.err
    echo "$c $env" >> gpurun_out/st256.jsonl
    [ $c = papers100m ] && break
  done
done
cat gpurun_out/st256.jsonl; grep check gpurun_out/st256.err
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-epoch > gpurun_out/b_st.json 2> gpurun_out/b_st.err
python -c "import json;d=json.load(open('gpurun_out/b_st.json'));print(d['value'],d['ms_per_step'],d['roofline']['avg_launch_us'],d['e2e']['value'])"
