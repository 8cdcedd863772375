python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; tail -1 gpurun_out/pytest_gpu.log
python tools/time_solve.py 5000:1072 50000:1072
python tools/trace_fac.py 50000 1072 2>&1 | grep "panel \["
