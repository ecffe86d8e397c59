set -x
nproc; free -g; df -h /dev/shm /tmp | cat; lscpu | grep -i "model name"; python -c "import numpy; numpy.show_config()" 2>&1 | grep -i -A3 "blas" | head -20
python -c "import __graft_entry__ as g; g.build()"
timeout 600 python bench.py --config papers100m --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/r2_p100m.json 2> gpurun_out/r2_p100m.err
tail -3 gpurun_out/r2_p100m.err; cat gpurun_out/r2_p100m.json
timeout 600 python bench.py --config mag240m --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/r2_mag.json 2> gpurun_out/r2_mag.err
tail -3 gpurun_out/r2_mag.err; cat gpurun_out/r2_mag.json
