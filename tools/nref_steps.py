"""Per trajectory position of bench.py's timed steps (C3, HyKKT): first-pass CG iterations, total CG
iterations, correction passes and the unrefined / refined omega -- shows which iterates need a second
correction pass.  Usage: [TAG=label] python tools/nref_steps.py"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, numpy as np
import bench
from paper_2403_15913_b200 import ckkt
dev = torch.device('cuda:0')
data = bench.build_inputs(50000, [0], dev)
pat, n, m = data['pat'], data['n'], data['m']
ctx = ckkt.Context(n, m, 0, pat.w_row, pat.w_col, pat.j_rowptr, pat.j_col, None, None, strategy=ckkt.CKKT_HYKKT, leaf=1072, device=0, stream=torch.cuda.current_stream().cuda_stream)
dx = torch.empty((1, n), dtype=torch.float64, device=dev); dy = torch.empty((1, m), dtype=torch.float64, device=dev)
T = data['w'].shape[0]
for k in range(3, 13):
    kk = k % T
    ctx.refactor(data['w'][kk], data['j'][kk], None, data['sig'][kk], None, None, None, None)
    rc, info = ctx.solve(data['r1'][kk], None, data['ra'][kk], None, dx, None, dy, None, want_info=True)
    i = info[0]
    print(os.environ.get('TAG',''), k, i['k_cg'], i['k_cg_total'], i['n_ref'], '%.3e %.3e' % (i['rel_res_unrefined'], i['rel_res']), flush=True)
