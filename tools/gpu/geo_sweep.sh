echo "restricted plans (surrogate)"
for s in "32 32" "32 64" "16 64" "64 32" "16 32" "32 16" "64 64"; do set -- $s; echo "BX $1 BY $2"; for f in poisson mass; do SG_GEOM_BX=$1 SG_GEOM_BY=$2 timeout 120 python tools/prof_one.py twisted 3 128 128 128 $f surrogate 16 2>&1 | tail -1 | grep -o "'geom_D', [0-9.]*" || echo fail; done; done
echo "ZB (full)"
for zb in 1 2 4 8 16 32; do echo "ZB $zb .."; for f in poisson mass; do SG_GEOM_ZB=$zb timeout 120 python tools/prof_one.py twisted 3 128 128 128 $f full 2>&1 | tail -1 | grep -o "'geom_D', [0-9.]*" || echo fail; done; done
