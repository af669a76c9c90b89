for d in 0 1 2 3 4 7; do echo "dbg $d"; SG_K7_DBG=$d python tools/prof_one.py twisted 3 128 128 128 mass surrogate 16 | tail -1 | grep -o "'interp_rows3', [0-9.]*"; done
