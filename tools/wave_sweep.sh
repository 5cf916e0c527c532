#!/bin/bash
# Wave-synchronised traversal on BASELINE configs[4] (48^3 x 96, nrhs 12):
# natural order vs patched+synchronised order for several patch budgets / slacks.
# Usage (GPU box): bash tools/wave_sweep.sh > gpurun_out/wave_sweep.txt 2>&1
D="96 48 48 48"
run() { echo "== $*"; env "$@" timeout 300 python tools/time_apply.py --dims $D --b 12 --dtypes c128 c64 --iters 10; }
run B200WD_WAVE_KB=0
run B200WD_WAVE_KB=16384
run B200WD_WAVE_KB=16384 B200WD_WAVE=0
run B200WD_WAVE_KB=8192
run B200WD_WAVE_KB=32768
run B200WD_WAVE_KB=16384 B200WD_WAVE_SLACK=1
run B200WD_WAVE_KB=16384 B200WD_WAVE_SLACK=4
