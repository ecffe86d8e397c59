# products-GAT: K-GEMM slice count re-sweep after the side-stream changes (FG_KGEMM_CHUNKS), interleaved
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r6x
for r in 1 2 3; do
for c in 0 24 48; do
FG_KGEMM_CHUNKS=$c timeout 600 python bench.py --config products-gat --steps 20 --warmup 5 --no-cpu-baseline --no-epoch > gpurun_out/r6x/b.json 2> gpurun_out/r6x/b.err
python -c "import json;d=json.load(open('gpurun_out/r6x/b.json'));print('chunks=$c', d['value'],d['ms_per_step'],d['e2e']['value'])"
done
done
