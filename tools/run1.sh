python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; tail -1 gpurun_out/pytest_gpu.log
CKKT_LIB_OVERRIDE=build_variants/t128_4/libckkt.so python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -1
echo "== cur"; python tools/time_solve.py 5000:1072 50000:1072
for v in t128_3 t128_4 t128_5; do echo "== $v"; CKKT_VERBOSE=1 CKKT_LIB_OVERRIDE=build_variants/$v/libckkt.so python tools/time_solve.py 5000:1072 50000:1072 2>&1 | grep -v "grids factor"; done
for tp in 2048 8192; do echo "== top $tp"; CKKT_TOP_PANEL=$tp python tools/time_solve.py 5000:1072 50000:1072; done
