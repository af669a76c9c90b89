timeout 900 python -m pytest -q -x -m gpu -p no:cacheprovider tests/test_gpu_fullsize.py tests/test_gpu_headline.py tests/test_gpu_multislab.py tests/test_gpu_assembly.py -k "not 2d_tiles" > gpurun_out/e2e_tests.log 2>&1; echo "tests rc $?"; tail -2 gpurun_out/e2e_tests.log
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu --no-sweep > gpurun_out/e2e_bench.log 2>&1; echo "bench rc $?"
python -c "
import json; d=json.loads(open('gpurun_out/e2e_bench.log').read().strip().splitlines()[-1]); print('value %.3e e2e %.3e' % (d['value'], d['e2e']['value']))"
