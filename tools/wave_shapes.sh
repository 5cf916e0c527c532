run() { echo "== $*"; env "${@:2}" timeout 300 python tools/time_apply.py --dims $1 --b 12 --dtypes c128 c64 --iters 10 2>&1 | grep frac; }
run "32 16 16 48" B200WD_WAVE_KB=0
run "32 16 16 16" B200WD_WAVE_KB=0
run "96 48 48 16" B200WD_WAVE_KB=0
run "96 48 48 16" B200WD_WAVE_KB=16384
run "96 48 48 16" B200WD_WAVE_KB=32768
run "96 48 48 16" B200WD_WAVE_KB=16384 B200WD_L2HINT=0
