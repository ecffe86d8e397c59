cd $GRAFT_REPO_ROOT
for ipt in 2 4 8 16; do
  FG_BM_IPT=$ipt timeout 600 python tools/chain_timing.py papers100m > gpurun_out/chain_ipt.txt 2>&1; echo "ipt=$ipt $(tail -1 gpurun_out/chain_ipt.txt)"
done
for ipt in 1 2 4; do
  FG_BM_IPT=$ipt timeout 600 python tools/chain_timing.py products > gpurun_out/chain_ipt.txt 2>&1; echo "products ipt=$ipt $(tail -1 gpurun_out/chain_ipt.txt)"
done
