#!/bin/bash
# Compare library variants on the BASELINE shapes (one GPU).
# usage: tools/variants_cmp.sh lib1.so lib2.so ...
for L in "$@"; do
  echo "=== $L"
  export B200WD_LIB=$L
  python tools/sweep_dirac.py --bs 4 8 12 16 32 --iters 30 2>&1 | grep -v "^#"
  python tools/sweep_dirac.py --dims 64 32 32 32 --bs 12 --dtypes c128 --parity 0 --iters 10 2>&1 | grep -v "^#"
  python tools/bench_schur.py 2>&1 | cut -c1-200
  python tools/bench_strong.py --dims 48 24 24 24 --dtypes c128,c64 --steps 20 2>&1 | cut -c150-260
done
