for bx in 32 16 64; do for by in 128 256 512; do echo "BX $bx BY $by"; for f in poisson mass; do SG_GEOM_BX=$bx SG_GEOM_BY=$by timeout 120 python tools/prof_one.py twisted 3 128 128 128 $f full 2>&1 | tail -1 | grep -o "'geom_D', [0-9.]*" || echo fail; done; done; done
echo surrogate
for by in 32 128 256; do echo "BX 32 BY $by"; for f in poisson mass; do SG_GEOM_BX=32 SG_GEOM_BY=$by timeout 120 python tools/prof_one.py twisted 3 128 128 128 $f surrogate 16 2>&1 | tail -1 | grep -o "'geom_D', [0-9.]*" || echo fail; done; done
