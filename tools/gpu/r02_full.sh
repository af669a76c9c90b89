# full -m gpu suite + default bench
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider --durations=10 > gpurun_out/r02_gputest.log 2>&1; echo "pytest rc $?"
tail -15 gpurun_out/r02_gputest.log
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/r02_bench.log 2> gpurun_out/r02_bench.err; echo "bench rc $?"
tail -c 400 gpurun_out/r02_bench.err
