echo "== base"; python tools/sweep_dirac.py --iters 50 --bs 4 8 16 32
for k in 1 2 4; do echo "== pf$k"; B200WD_LIB=build_variants/lib_pf$k.so python tools/sweep_dirac.py --iters 50 --bs 4 8 16 32; done
