# T-stream tuning sweep: B200WD_TS_CFG="NB,LY,S,NCH,PF" per (dtype, nrhs)
dt=$1; b=$2; shift 2
for c in "$@"; do echo "cfg $c"; B200WD_TS_CFG=$c timeout 120 python tools/sweep_dirac.py --dtypes $dt --bs $b --iters 20 2>&1 | grep frac; done
