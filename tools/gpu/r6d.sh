# lane kernels: FMUL2 epilogue + fixed staging offsets (new2) vs fanout-5 fast path (new); MAG GEMM formulations
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r6d
( timeout 900 python -m pytest tests/test_gpu_aggregate.py tests/test_gpu_fullscale.py -m gpu -x -q ) > gpurun_out/r6d/t.log 2>&1
tail -1 gpurun_out/r6d/t.log; grep -E "^E " gpurun_out/r6d/t.log | head
L=paper_2207_14696_b200/libfgb200.so
for cfg in mag240m papers100m products; do
for v in new new2 new new2; do
cp abtmp/libfgb200_$v.so $L
timeout 600 python tools/fused_bench.py --config $cfg --iters 30 > gpurun_out/r6d/fb_${cfg}_$v.txt 2>&1
echo "$cfg $v: $(tail -1 gpurun_out/r6d/fb_${cfg}_$v.txt | python -c 'import json,sys;d=json.loads(sys.stdin.read());print(d["avg_us"],d["min_us"],d["frac"])')"
done
done
cp abtmp/libfgb200_new2.so $L
timeout 600 python tools/gemm_probe.py > gpurun_out/r6d/gemm_probe.txt 2>&1; cat gpurun_out/r6d/gemm_probe.txt
