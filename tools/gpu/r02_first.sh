# round-2 first GPU pass: full -m gpu suite, then the default bench
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/r02_gputest.log 2>&1; echo "pytest rc $?"
tail -5 gpurun_out/r02_gputest.log
timeout 600 python bench.py --steps 5 --warmup 3 > gpurun_out/r02_bench.log 2>&1; echo "bench rc $?"
tail -c 3000 gpurun_out/r02_bench.log
