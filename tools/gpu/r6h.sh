# VQ lane kernel: 512 threads x 112 registers with paired 5-pick destinations (FG_VQ_LANE_NT=512) vs 1024 threads
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r6h
for cfg in mag240m products; do
for nt in 1024 512 1024 512; do
FG_VQ_LANE_NT=$nt timeout 600 python tools/fused_bench.py --config $cfg --iters 40 --check > gpurun_out/r6h/fb_${cfg}_$nt.txt 2>&1
echo "$cfg $nt: $(grep check gpurun_out/r6h/fb_${cfg}_$nt.txt | cut -c1-80) $(tail -1 gpurun_out/r6h/fb_${cfg}_$nt.txt | python -c 'import json,sys;d=json.loads(sys.stdin.read());print(d["avg_us"],d["min_us"],d["frac"])')"
done
done
