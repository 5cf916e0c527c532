#!/bin/bash
# Cost of the patched (TILED) order and of the wave synchronisation on an
# L2-resident lattice (no DRAM effect): natural vs forced TILED, with / without waves.
run() { echo "== $*"; env "${@:2}" timeout 300 python tools/time_apply.py --dims $1 --b 12 16 --dtypes c128 c64 --iters 20 2>&1 | grep frac; }
run "32 16 16 16" B200WD_WAVE_KB=0
run "32 16 16 16" B200WD_SLICE_KB=1 B200WD_WAVE_KB=2048 B200WD_WAVE=0
run "32 16 16 16" B200WD_SLICE_KB=1 B200WD_WAVE_KB=2048
run "32 16 16 16" B200WD_SLICE_KB=1 B200WD_WAVE_KB=2048 B200WD_WAVE_SLACK=8
run "32 16 16 16" B200WD_SLICE_KB=1 B200WD_WAVE_KB=2048 B200WD_L2HINT=0
