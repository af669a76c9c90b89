set -x
timeout 900 python -m pytest tests/test_gpu_multislab.py tests/test_gpu_surrogate.py tests/test_gpu_assembly.py tests/test_gpu_headline.py -q -x -p no:cacheprovider -m gpu > gpurun_out/r02_slab_tests.log 2>&1; echo "tests rc $?"
tail -3 gpurun_out/r02_slab_tests.log
timeout 900 python tools/slab_cost.py > gpurun_out/r02_slab_cost.txt 2>&1; echo "rc $?"
cat gpurun_out/r02_slab_cost.txt
SG_SLABS=8 timeout 600 python tools/slab_breakdown.py > gpurun_out/r02_slab_breakdown.txt 2>&1
grep -A3 "surrogate whole" gpurun_out/r02_slab_breakdown.txt
