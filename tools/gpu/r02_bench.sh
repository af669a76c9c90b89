set -x
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/r02_bench.log 2> gpurun_out/r02_bench.err; echo "bench rc $?"
tail -c 600 gpurun_out/r02_bench.err
python bench.py --gpus 2 --steps 1 --warmup 1 --no-cpu > gpurun_out/r02_bench_g2.log 2>&1; echo "g2 rc $?"; tail -3 gpurun_out/r02_bench_g2.log
