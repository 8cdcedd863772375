CKKT_LIB_OVERRIDE=build_variants/buggy/libckkt.so python -m pytest tests/test_gpu_parity.py -x -q -k "wider" 2>&1 | tail -3
