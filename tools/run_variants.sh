python -m pytest tests/test_gpu_dirac.py -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
tail -2 gpurun_out/pytest_gpu.log
echo "== table"; python tools/sweep_dirac.py --iters 50
