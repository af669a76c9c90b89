# canonical interior tables + 2D fragment reuse: parity subset, then configs 2/4 device times
timeout 1200 python -m pytest -q -x -m gpu -p no:cacheprovider tests/test_gpu_assembly.py tests/test_gpu_surrogate.py tests/test_gpu_headline.py > gpurun_out/canon_tests.log 2>&1; echo "tests rc $?"; tail -3 gpurun_out/canon_tests.log
for f in poisson mass; do python tools/prof_one.py annulus 3 512 512 $f full | tail -1; python tools/prof_one.py annulus 3 512 512 $f surrogate 16 | tail -1; done
python tools/prof_one.py sinmap 3 1024 1024 biharmonic full | tail -1; python tools/prof_one.py sinmap 3 1024 1024 biharmonic surrogate 32 | tail -1
python tools/prof_one.py twisted 3 128 128 128 poisson full | tail -1
