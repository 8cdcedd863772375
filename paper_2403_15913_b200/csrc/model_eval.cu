// Distillation-column model evaluation on the GPU ("GPU model evaluation
// (ExaModels-style AD of distillation W, J) ... completes the per-iteration GPU pipeline").
//
// The NLP of P:489-530 (reading A, R12/R14): per stage t the 67 variables x_1..x_32, y_1..y_32,
// u, L, V; 66 equality rows (stage 0: 32 initial conditions, L-row, V-row, 32 VLE rows; stage t >= 1:
// L-row, V-row, 32 VLE rows, 32 implicit-Euler balances).  One warp per stage, lane k = tray k: the
// Jacobian values J = dg/dv in the CSR order of inputs/distillation.build_pattern (rows scaled by
// row_scale), the Hessian of the Lagrangian W = obj_scale grad^2 f + sum_r lam_r row_scale_r grad^2 g_r
// in the pattern's sorted lower order, the scaled residual c and the scaled objective gradient — the
// derivative formulas of SURVEY §8(d) (the table "Generator derivative formulas"), the same expressions
// the host generator evaluates, each entry once (no atomics).
#include <cuda_runtime.h>

#include <cmath>

#include "../../include/ckkt.h"

namespace {

constexpr int NV = 67, NR = 66, NT = 32;
constexpr int OX = 0, OY = 32, OU = 64, OL = 65, OV = 66;

struct Dev {
  double alpha, D, F, w_x, rho, dt, x_f, xbar1, ubar;
  int feed;  // 0-based feed tray
  double M[NT];
};

__device__ __forceinline__ double vle(const Dev& p, double x) { return p.alpha * x / (1.0 + (p.alpha - 1.0) * x); }
__device__ __forceinline__ double vle_d1(const Dev& p, double x) {
  const double q = 1.0 + (p.alpha - 1.0) * x;
  return p.alpha / (q * q);
}
__device__ __forceinline__ double vle_d2(const Dev& p, double x) {
  const double q = 1.0 + (p.alpha - 1.0) * x;
  return -2.0 * p.alpha * (p.alpha - 1.0) / (q * q * q);
}

// one warp per (stage t, instance b); lane k = tray k
__global__ void k_distillation_eval(int N, int B, Dev p, const double* __restrict__ xbar0, const double* __restrict__ v,
                                    const double* __restrict__ lam, const double* __restrict__ rs, double sf,
                                    double* __restrict__ jv, double* __restrict__ wv, double* __restrict__ c,
                                    double* __restrict__ gf) {
  const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, k = threadIdx.x & 31;
  if (gw >= (N + 1) * B) return;
  const int t = gw % (N + 1), b = gw / (N + 1);
  const int64_t n = (int64_t)NV * (N + 1), m = (int64_t)NR * (N + 1);
  const int64_t nnzj = 288ll * N + 100, nnzw = 96ll * N + 32;
  const double* vb = v + b * n;
  const double* vs = vb + (int64_t)NV * t;
  const double x = vs[OX + k], y = vs[OY + k], u = vs[OU], Lf = vs[OL], V = vs[OV];
  const int64_t r0 = (int64_t)NR * t;  // first row of the stage
  const double* rsb = rs ? rs + b * m : nullptr;
  auto RS = [&](int64_t r) { return rsb ? rsb[r] : 1.0; };
  const double* lb = lam ? lam + b * m : nullptr;
  if (t == 0) {
    // rows: IC (32), L-row, V-row, VLE (32); J entries: IC 1 | L-row [u, L] | V-row [L, V] | VLE [x_k, y_k]
    if (jv) {
      double* J = jv + b * nnzj;
      J[k] = 1.0 * RS(k);
      if (k == 0) {
        J[32] = -p.D * RS(32);
        J[33] = 1.0 * RS(32);
        J[34] = -1.0 * RS(33);
        J[35] = 1.0 * RS(33);
      }
      J[36 + 2 * k] = -vle_d1(p, x) * RS(34 + k);
      J[37 + 2 * k] = 1.0 * RS(34 + k);
    }
    if (c) {
      double* C = c + b * m;
      C[k] = (x - xbar0[k]) * RS(k);
      if (k == 0) {
        C[32] = (Lf - u * p.D) * RS(32);
        C[33] = (V - Lf - p.D) * RS(33);
      }
      C[34 + k] = (y - vle(p, x)) * RS(34 + k);
    }
    if (wv) {  // (x_k, x_k): VLE curvature only (no objective term at t = 0)
      const double l = lb ? lb[34 + k] * RS(34 + k) : 0.0;
      wv[b * nnzw + k] = -l * vle_d2(p, x);
    }
    if (gf) {
      double* G = gf + b * n;
      G[OX + k] = 0.0;
      G[OY + k] = 0.0;
      if (k < 3) G[OU + k] = 0.0;
    }
    return;
  }
  // ---- stage t >= 1
  const double* ps = vs - NV;  // previous stage
  const double xp = ps[OX + k];
  const double S = p.F + Lf, dt = p.dt;
  // neighbours along the column (lane shuffles)
  const double x_dn = __shfl_up_sync(0xffffffffu, x, 1);      // x_{k-1}
  const double y_up = __shfl_down_sync(0xffffffffu, y, 1);    // y_{k+1}
  const double Mk = p.M[k];
  if (jv) {
    double* J = jv + b * nnzj + 100 + 288ll * (t - 1);
    const int64_t rL = r0, rV = r0 + 1, rvle = r0 + 2 + k, rbal = r0 + 34 + k;
    if (k == 0) {
      J[0] = -p.D * RS(rL);
      J[1] = 1.0 * RS(rL);
      J[2] = -1.0 * RS(rV);
      J[3] = 1.0 * RS(rV);
    }
    J[4 + 2 * k] = -vle_d1(p, x) * RS(rvle);
    J[5 + 2 * k] = 1.0 * RS(rvle);
    const double sc = RS(rbal);
    if (k == 0) {  // condenser: [x1-, x1, y2, V]
      double* Jb = J + 68;
      Jb[0] = (-1.0 / dt) * sc;
      Jb[1] = (1.0 / dt + V / Mk) * sc;
      Jb[2] = (-V / Mk) * sc;
      Jb[3] = (-(y_up - x) / Mk) * sc;
    } else if (k < NT - 1) {  // trays 2..31: [x-, x_{k-1}, x_k, y_k, y_{k+1}, L, V]
      double* Jb = J + 72 + 7 * (k - 1);
      double c_prev, c_self;
      if (k == p.feed) {
        c_prev = -Lf / Mk;
        c_self = 1.0 / dt + S / Mk;
      } else {
        const double flow = (k < p.feed) ? Lf : S;
        c_prev = -flow / Mk;
        c_self = 1.0 / dt + flow / Mk;
      }
      Jb[0] = (-1.0 / dt) * sc;
      Jb[1] = c_prev * sc;
      Jb[2] = c_self * sc;
      Jb[3] = (V / Mk) * sc;
      Jb[4] = (-V / Mk) * sc;
      Jb[5] = (-(x_dn - x) / Mk) * sc;
      Jb[6] = ((y - y_up) / Mk) * sc;
    } else {  // reboiler: [x32-, x31, x32, y32, L, V]
      double* Jb = J + 72 + 7 * (NT - 2);
      Jb[0] = (-1.0 / dt) * sc;
      Jb[1] = (-S / Mk) * sc;
      Jb[2] = (1.0 / dt + (p.F - p.D) / Mk) * sc;
      Jb[3] = (V / Mk) * sc;
      Jb[4] = (-x_dn / Mk) * sc;
      Jb[5] = (y / Mk) * sc;
    }
  }
  if (c) {
    double* C = c + b * m + r0;
    if (k == 0) {
      C[0] = (Lf - u * p.D) * RS(r0);
      C[1] = (V - Lf - p.D) * RS(r0 + 1);
    }
    C[2 + k] = (y - vle(p, x)) * RS(r0 + 2 + k);
    double xd;  // material balance right-hand side (reboiler reading R12)
    if (k == 0) xd = V * (y_up - x) / Mk;
    else if (k < p.feed) xd = (Lf * (x_dn - x) - V * (y - y_up)) / Mk;
    else if (k == p.feed) xd = (p.F * p.x_f + Lf * x_dn - S * x - V * (y - y_up)) / Mk;
    else if (k < NT - 1) xd = (S * (x_dn - x) - V * (y - y_up)) / Mk;
    else xd = (S * x_dn - (p.F - p.D) * x - V * y) / Mk;
    C[34 + k] = ((x - xp) / dt - xd) * RS(r0 + 34 + k);
  }
  if (wv) {
    // multipliers (scaled): VLE rows lv_k, balance rows lb_k (lane k), neighbours by shuffles
    const double lvk = lb ? lb[r0 + 2 + k] * RS(r0 + 2 + k) : 0.0;
    const double lbk = lb ? lb[r0 + 34 + k] * RS(r0 + 34 + k) : 0.0;
    const double q_k = lbk / Mk;                                     // lb_k / M_k
    const double q_up = __shfl_down_sync(0xffffffffu, q_k, 1);      // lb_{k+1} / M_{k+1}
    const double q_dn = __shfl_up_sync(0xffffffffu, q_k, 1);        // lb_{k-1} / M_{k-1}
    const double q_0 = __shfl_sync(0xffffffffu, q_k, 0);            // lb_0 / M_0
    double* W = wv + b * nnzw + 32 + 96ll * (t - 1);
    double dxx = -lvk * vle_d2(p, x);
    if (k == 0) dxx += 2.0 * p.w_x * sf;
    W[k] = dxx;                                   // (x_k, x_k), k = 0..31
    if (k == 0) W[32] = 2.0 * p.rho * sf;         // (u, u)
    if (k < NT - 1) {                             // (L, x_k), k = 0..30
      double d = 0.0 + (-q_up);
      if (k >= 1) d += q_k;
      W[33 + k] = d;
    }
    if (k == 0) W[64] = q_0;                      // (V, x_1)
    if (k >= 1) {                                 // (V, y_k), k = 1..31
      double d = 0.0;
      if (k == 1) d += -q_0;
      d += q_k;
      if (k >= 2) d += -q_dn;
      W[65 + (k - 1)] = d;
    }
  }
  if (gf) {
    double* G = gf + b * n + (int64_t)NV * t;
    G[OX + k] = (k == 0) ? sf * (2.0 * p.w_x * (x - p.xbar1)) : 0.0;
    G[OY + k] = 0.0;
    if (k == 0) G[OU] = sf * (2.0 * p.rho * (u - p.ubar));
    if (k == 1) G[OL] = 0.0;
    if (k == 2) G[OV] = 0.0;
  }
}

}  // namespace

extern "C" ckkt_status ckkt_distillation_eval(int32_t N, int32_t batch, const ckkt_distillation_params* prm,
                                              const double* xbar0, const double* v, const double* lam,
                                              const double* row_scale, double obj_scale, double* j_val,
                                              double* w_val, double* c, double* grad_f, void* stream) {
  if (N < 1 || batch < 1 || !prm || !v || (c && !xbar0) || !(prm->horizon > 0.0) || prm->feed_tray < 2 ||
      prm->feed_tray > NT - 1 || !std::isfinite(obj_scale))
    return CKKT_INVALID_ARG;
  Dev p;
  p.alpha = prm->alpha;
  p.D = prm->D;
  p.F = prm->F;
  p.w_x = prm->w_x;
  p.rho = prm->rho;
  p.dt = prm->horizon / N;
  p.x_f = prm->x_f;
  p.xbar1 = prm->xbar1;
  p.ubar = prm->ubar;
  p.feed = prm->feed_tray - 1;
  for (int k = 0; k < NT; ++k) {
    if (!(prm->M[k] > 0.0)) return CKKT_INVALID_ARG;
    p.M[k] = prm->M[k];
  }
  const int64_t warps = (int64_t)(N + 1) * batch;
  const unsigned blocks = (unsigned)((warps * 32 + 255) / 256);
  k_distillation_eval<<<blocks, 256, 0, (cudaStream_t)stream>>>(N, batch, p, xbar0, v, lam, row_scale, obj_scale,
                                                                j_val, w_val, c, grad_f);
  return cudaGetLastError() == cudaSuccess ? CKKT_OK : CKKT_CUDA_ERROR;
}
