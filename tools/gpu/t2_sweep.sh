for t in 24 48 66 96 131; do echo "T2 $t"; for f in poisson mass; do SG_T2_RESTR=$t python tools/prof_one.py twisted 3 128 128 128 $f surrogate 16 | tail -1 | python -c "
import sys,ast
l=sys.stdin.read().strip(); tot=float(l[1:l.index(',')]); print(round(tot,3))"; done; done
echo config3; for t in 24 48 66; do SG_T2_RESTR=$t python tools/prof_one.py twisted 2 64 64 64 poisson surrogate 8 | tail -1 | cut -c1-20; done
