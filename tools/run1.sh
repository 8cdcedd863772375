python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; tail -2 gpurun_out/pytest_gpu.log
for v in prev acq; do echo "== $v"; CKKT_LIB_OVERRIDE=build_variants/$v/libckkt.so python tools/time_solve.py 5000:1072 50000:1072; done
echo "== cur"; python tools/time_solve.py 5000:1072 50000:1072
