# K4 3D: correctness subset, then device times of config-5 full assemblies
timeout 900 python -m pytest -q -x -m gpu -p no:cacheprovider tests/test_gpu_assembly.py tests/test_gpu_surrogate.py tests/test_gpu_headline.py -k "golden or rows3 or c5s48 or zero or slab or c3_" > gpurun_out/k4_tests.log 2>&1; echo "tests rc $?"; tail -3 gpurun_out/k4_tests.log
for f in poisson mass; do python tools/prof_one.py twisted 3 128 128 128 $f full | tail -1; python tools/prof_one.py twisted 3 128 128 128 $f surrogate 16 | tail -1; done
