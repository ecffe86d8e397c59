# MAG lane kernel bisect: FMUL2 epilogue (A), staging-first smem layout (B), A + hoisted store predicate (C) vs current (new)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r6f
L=paper_2207_14696_b200/libfgb200.so
cp $L abtmp/libfgb200_cur.so
for cfg in mag240m; do
for v in new A B C new A B C; do
cp abtmp/libfgb200_$v.so $L
timeout 600 python tools/fused_bench.py --config $cfg --iters 40 > gpurun_out/r6f/fb_${cfg}_$v.txt 2>&1
echo "$cfg $v: $(tail -1 gpurun_out/r6f/fb_${cfg}_$v.txt | python -c 'import json,sys;d=json.loads(sys.stdin.read());print(d["avg_us"],d["min_us"],d["frac"])')"
done
done
cp abtmp/libfgb200_cur.so $L
