for v in base nopf minb4 minb5; do echo "== $v"; CKKT_LIB_OVERRIDE=build_variants/$v/libckkt.so python tools/time_solve.py 5000:1072 50000:1072; done
echo "== cur"; python tools/time_solve.py 5000:1072 50000:1072
