# polynomial-map geometry (K3 without the quotient rule): parity subset, then config-5 / 4 / 2 geom_D times
timeout 1200 python -m pytest -q -x -m gpu -p no:cacheprovider tests/test_gpu_assembly.py tests/test_gpu_surrogate.py tests/test_gpu_headline.py tests/test_gpu_fullsize.py > gpurun_out/geo_tests.log 2>&1; echo "tests rc $?"; tail -3 gpurun_out/geo_tests.log
for f in poisson mass; do python tools/prof_one.py twisted 3 128 128 128 $f full | tail -1; SG_GEO_QUOTIENT=1 python tools/prof_one.py twisted 3 128 128 128 $f full | tail -1; done
python tools/prof_one.py sinmap 3 1024 1024 biharmonic full | tail -1
