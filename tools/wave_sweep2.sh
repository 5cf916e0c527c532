#!/bin/bash
# configs[4] (48^3 x 96, nrhs 12) natural vs wave-synchronised order, early-release build
D="96 48 48 48"
run() { echo "== $*"; env "$@" timeout 300 python tools/time_apply.py --dims $D --b 12 --dtypes c128 --iters 10 | grep frac; }
run B200WD_WAVE_KB=0
run B200WD_WAVE=1 B200WD_WAVE_KB=16384 B200WD_WAVE_SLACK=2
run B200WD_WAVE=1 B200WD_WAVE_KB=16384 B200WD_WAVE_SLACK=3
run B200WD_WAVE=1 B200WD_WAVE_KB=24576 B200WD_WAVE_SLACK=2
run B200WD_WAVE=1 B200WD_WAVE_KB=8192 B200WD_WAVE_SLACK=4
run B200WD_WAVE=0 B200WD_WAVE_KB=16384
