for cfg in "2,4" "4,4" "4,3" "2,2" "2,3"; do echo "== c64 RING_CFG=$cfg"; B200WD_TSTREAM=0 B200WD_RING2_S=0 B200WD_RING_CFG=$cfg python tools/sweep_dirac.py --bs 8 12 16 32 --dtypes c64 --iters 30 2>&1 | grep -v "^#"; done
for cfg in "2,3" "2,4" "4,4"; do echo "== c128 RING_CFG=$cfg"; B200WD_RING_CFG=$cfg python tools/sweep_dirac.py --bs 8 16 --dtypes c128 --iters 30 2>&1 | grep -v "^#"; done
