# round-2 measurement pass: default bench line, then the ncu launch list of one bench step
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/r02_bench.log 2> gpurun_out/r02_bench.err; echo "bench rc $?"
CMD="python bench.py --steps 1 --warmup 1 --no-cpu --no-sweep --no-e2e"
$CMD > gpurun_out/r02_launch_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02_launches.csv $CMD > gpurun_out/r02_launch_ncu.log 2>&1
echo "ncu rc $?"
