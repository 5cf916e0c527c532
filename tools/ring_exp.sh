#!/bin/bash
# Ring-kernel experiment variants (build_variants/lib_exp*.so, B200WD_RING_EXP bits;
# timing only -- bits 0/1/2/4 give wrong results): what bounds the tile ingress.
# usage: tools/ring_exp.sh [names...]   (default: every build_variants/lib_exp*.so)
cd "$(dirname "$0")/.."
export B200WD_TSTREAM=0 B200WD_RING2_S=0
names=${@:-base $(ls build_variants | sed -n 's/^lib_\(exp[0-9a-z]*\)\.so$/\1/p')}
for v in $names; do
  if [ "$v" = base ]; then unset B200WD_LIB; else export B200WD_LIB=$PWD/build_variants/lib_$v.so; fi
  echo "== $v"
  python tools/time_apply.py --dims 32 16 16 16 --b 8 16 --dtypes c128 --iters 30 | sed 's/dims=.*clov=0//'
  python tools/time_apply.py --dims 32 16 16 16 --b 16 32 --dtypes c64 --iters 30 | sed 's/dims=.*clov=0//'
done
