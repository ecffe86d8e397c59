# GAT side-stream operands (tests + bench) and lane-kernel fanout-5 fast path A/B (fused_bench, base vs new lib)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r6c
( timeout 900 python -m pytest tests/test_gpu_gat.py tests/test_gpu_aggregate.py -m gpu -x -q ) > gpurun_out/r6c/t.log 2>&1
tail -1 gpurun_out/r6c/t.log; grep -E "^E " gpurun_out/r6c/t.log | head
for r in 1 2; do
timeout 900 python bench.py --config products-gat --steps 30 --warmup 5 --no-cpu-baseline --no-epoch > gpurun_out/r6c/b_gat$r.json 2> gpurun_out/r6c/b_gat$r.err
python -c "import json;d=json.load(open('gpurun_out/r6c/b_gat$r.json'));print('gat', d['value'],d['ms_per_step'],d['e2e']['value'])"
done
L=paper_2207_14696_b200/libfgb200.so
for cfg in mag240m papers100m; do
for v in base new base new; do
cp abtmp/libfgb200_$v.so $L
timeout 600 python tools/fused_bench.py --config $cfg --iters 30 > gpurun_out/r6c/fb_${cfg}_$v.txt 2>&1
echo "$cfg $v: $(tail -1 gpurun_out/r6c/fb_${cfg}_$v.txt | cut -c1-300)"
done
done
