// CG vector kernels (K4 of SURVEY §2C): fused, vectorised, deterministic.
//
// Alg. 1 with the paper's fusions: r -= alpha Ap fused with r.r, and
// x += alpha p; p = r + beta p (fused with p.p).  The paper's separate p.Ap kernel is folded
// into the operator as the element energy (ax_lines.cuh energy_finish).  alpha and beta never leave
// the device: every kernel reads the reduced scalars from CgScalars and computes them
// itself, so an iteration has no host round trip and can be captured in a CUDA graph.
// Reductions: fp64 per thread -> warp shuffle -> CTA -> one partial per CTA; the last CTA
// to finish (atomic ticket) sums the partials in CTA order, so results are deterministic
// for a fixed grid.  With P > 1 the local sum is allreduced (NCCL) before use.
#pragma once
#include <cstdint>

#include <cooperative_groups.h>

#include "common.cuh"  // CgScalars

namespace hbk {

constexpr int VEC_BLOCK = 512;

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// CTA sum; result valid in thread 0
__device__ __forceinline__ double block_sum(double v) {
  __shared__ double s_w[VEC_BLOCK / 32];
  v = warp_sum(v);
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  if (lane == 0) s_w[w] = v;
  __syncthreads();
  double r = 0.0;
  if (w == 0) {
    r = lane < VEC_BLOCK / 32 ? s_w[lane] : 0.0;
    r = warp_sum(r);
  }
  return r;
}

// Writes the CTA partial; returns true in thread 0 of the last CTA, with the ordered total.
__device__ __forceinline__ bool finish_reduction(double v, double* partials, uint32_t* ticket, double* total) {
  __shared__ bool s_last;
  double b = block_sum(v);
  if (threadIdx.x == 0) {
    partials[blockIdx.x] = b;
    __threadfence();
    uint32_t tk = atomicAdd(ticket, 1u);
    s_last = (tk == gridDim.x - 1);
  }
  __syncthreads();
  if (!s_last) return false;
  // last CTA: ordered sum of all partials
  __threadfence();
  double acc = 0.0;
  for (int b2 = threadIdx.x; b2 < (int)gridDim.x; b2 += VEC_BLOCK) acc += ((volatile double*)partials)[b2];
  // deterministic: fixed strided assignment + fixed tree
  acc = block_sum(acc);
  if (threadIdx.x == 0) {
    *total = acc;
    *ticket = 0u;
  }
  return threadIdx.x == 0;
}

// r = b; p = z (= b, or M^-1 b with the Jacobi preconditioner); x = 0; Ap = lam_init * p;
// global r.r -> rr_new (and r.z -> rz), CTA partials of p.p -> pp_part (fused path)
__global__ void __launch_bounds__(VEC_BLOCK)
cg_init(const double* __restrict__ b, double* __restrict__ x, double* __restrict__ r,
        double* __restrict__ p, double* __restrict__ Ap, int64_t n, double lam_init,
        double* partials, CgScalars* s, double* pp_part, const double* __restrict__ invd) {
  double acc = 0.0, acc_rz = 0.0, acc_pp = 0.0;
  for (int64_t l = (int64_t)blockIdx.x * VEC_BLOCK + threadIdx.x; l < n; l += (int64_t)gridDim.x * VEC_BLOCK) {
    const double v = b[l];
    const double z = invd ? v * invd[l] : v;
    r[l] = v; p[l] = z; x[l] = 0.0; Ap[l] = lam_init * z;
    acc = fma(v, v, acc);
    acc_rz = fma(v, z, acc_rz);
    acc_pp = fma(z, z, acc_pp);
  }
  if (pp_part) {  // the CTA partials of p.p for the fused update's first p.Ap
    const double bs = block_sum(acc_pp);
    if (threadIdx.x == 0) pp_part[blockIdx.x] = bs;
    __syncthreads();
  }
  if (invd) {  // r.z: ordered two-level sum (its own slice of the partials buffer)
    double t;
    if (finish_reduction(acc_rz, partials, &s->ticket, &t)) s->rz = t;
    __syncthreads();
  }
  double tot;
  if (finish_reduction(acc, partials + gridDim.x, &s->ticket_e, &tot)) {
    s->rr_new = tot;        // allreduced for P > 1
    if (!invd) s->rz = tot;
    s->pp = tot;            // local p.p for the P > 1 path (no preconditioner there: p = r)
    s->e_acc = 0.0;
    s->it = 0;
    s->flags = 0;
  }
}

// One GPU: the operator left one energy partial per CTA (e_part[0..n_part)); every CTA of
// this kernel reduces them in the same fixed order, so p.Ap = sum + lambda p.p is identical
// everywhere without an extra kernel or a fence/atomic in the operator.  Then alpha = rr / p.Ap,
// x += alpha p, r -= alpha Ap with the CTA partials of r.r; the last CTA rotates rr <- r_j.r_j,
// records the history, publishes p.Ap and leaves r_{j+1}.r_{j+1} in rr_loc for the p update.
__global__ void __launch_bounds__(VEC_BLOCK)
cg_update_xr_e(double* __restrict__ x, const double* __restrict__ p, double* __restrict__ r,
               const double* __restrict__ Ap, int64_t n, const double* __restrict__ e_part, int n_part,
               double lam_pp, double* partials, CgScalars* s, double* hist) {
  __shared__ double s_pAp;
  double ev = 0.0;
  for (int b = threadIdx.x; b < n_part; b += VEC_BLOCK) ev += e_part[b];
  ev = block_sum(ev);
  const double rr = s->rr_new;  // r_j.r_j
  if (threadIdx.x == 0) s_pAp = ev + lam_pp * s->pp;
  __syncthreads();
  const double pAp = s_pAp;
  const double alpha = (pAp != 0.0) ? rr / pAp : 0.0;  // c15 guard
  double acc = 0.0;
  const int64_t n2 = n >> 1;
  double2* x2 = reinterpret_cast<double2*>(x);
  double2* r2 = reinterpret_cast<double2*>(r);
  const double2* p2 = reinterpret_cast<const double2*>(p);
  const double2* a2 = reinterpret_cast<const double2*>(Ap);
  for (int64_t l = (int64_t)blockIdx.x * VEC_BLOCK + threadIdx.x; l < n2; l += (int64_t)gridDim.x * VEC_BLOCK) {
    double2 xv = x2[l], pv = p2[l], rv = r2[l], av = a2[l];
    xv.x = fma(alpha, pv.x, xv.x); xv.y = fma(alpha, pv.y, xv.y);
    rv.x = fma(-alpha, av.x, rv.x); rv.y = fma(-alpha, av.y, rv.y);
    x2[l] = xv; r2[l] = rv;
    acc = fma(rv.x, rv.x, acc); acc = fma(rv.y, rv.y, acc);
  }
  if ((n & 1) && blockIdx.x == 0 && threadIdx.x == 0) {
    const int64_t l = n - 1;
    x[l] = fma(alpha, p[l], x[l]);
    double rv = fma(-alpha, Ap[l], r[l]);
    r[l] = rv;
    acc = fma(rv, rv, acc);
  }
  double tot;
  if (finish_reduction(acc, partials, &s->ticket, &tot)) {
    s->pAp = pAp;
    s->rr = rr;
    if (hist) hist[s->it] = rr;
    s->rr_loc = tot;
  }
}

// Tolerance-mode loop test folded into the fused vector update (the WHILE body's last kernel
// publishes the scalars anyway): Alg. 1 line 6 (while r.r > eps), the iteration cap and
// the breakdown check (p.Ap <= 0 or non-finite) set the WHILE node's condition -- one launch
// per trip fewer than a separate cg_continue kernel.
struct CondTest {
  cudaGraphConditionalHandle h;
  double eps;
  int32_t max_iters;
  int32_t on;
};
__device__ __forceinline__ void cond_test(const CondTest& ct, CgScalars* s, double pAp, double rr_new, int32_t it) {
  bool go = rr_new > ct.eps && it < ct.max_iters;
  if (!(pAp > 0.0) || !isfinite(pAp) || !isfinite(rr_new)) {
    s->flags |= 1;
    go = false;
  }
  cudaGraphSetConditional(ct.h, go ? 1u : 0u);
}

// One GPU, whole vector update of an iteration in one cooperative kernel (grid barrier
// instead of a kernel boundary): p.Ap = sum(e_part) + lambda sum(pp_part) (deterministic,
// every CTA alike); x += alpha p, r -= alpha Ap, CTA partial of r.r; grid barrier; every CTA
// sums the r.r partials in CTA order -> beta; p = r + beta p, Ap = lambda p, CTA partial of
// p.p (consumed by the next iteration's p.Ap).  r and p are re-read after the barrier from L2
// when the vectors fit it.  CTA 0 publishes the scalars (pAp, rr, rr_new, history, j).
// (single-item form; the batched cg_update_fused below is used for vectors that fit L2)
// COND: the tolerance-mode instance, which also runs the loop test and sets the WHILE node's
// condition (ncu does not profile kernels that can set conditional handles, so the fixed-mode
// graph uses the COND = false instance)
template <bool COND>
__global__ void __launch_bounds__(VEC_BLOCK)
cg_update_fused0(double* __restrict__ x, double* __restrict__ p, double* __restrict__ r, double* __restrict__ Ap,
                int64_t n, const double* __restrict__ e_part, int n_epart, double* pp_part, double lam_pp,
                double lam_init, double* rr_part, CgScalars* s, double* hist, const double* __restrict__ invd,
                double* rz_part, CondTest ct) {
  __shared__ double s_b[3];
  pdl_wait();
  // ---- p.Ap and alpha (identical in every CTA)
  double ev = 0.0, pv_ = 0.0;
  for (int b = threadIdx.x; b < n_epart; b += VEC_BLOCK) ev += e_part[b];
  for (int b = threadIdx.x; b < (int)gridDim.x; b += VEC_BLOCK) pv_ += pp_part[b];
  ev = block_sum(ev);
  __syncthreads();
  pv_ = block_sum(pv_);
  const double rr = s->rr_new;             // r_j.r_j
  const double rho = invd ? s->rz : rr;     // r_j.z_j (PCG) or r_j.r_j (CG)
  if (threadIdx.x == 0) s_b[0] = ev + lam_pp * pv_;
  __syncthreads();
  const double pAp = s_b[0];
  const double alpha = (pAp != 0.0) ? rho / pAp : 0.0;  // c15 guard
  // ---- x, r update + r.r (+ r.z)
  const int64_t n2 = n >> 1;
  const int64_t stride = (int64_t)gridDim.x * VEC_BLOCK;
  double acc = 0.0, acc_rz = 0.0;
  const double2* d2 = reinterpret_cast<const double2*>(invd);
  {
    double2* x2 = reinterpret_cast<double2*>(x);
    double2* r2 = reinterpret_cast<double2*>(r);
    const double2* p2 = reinterpret_cast<const double2*>(p);
    const double2* a2 = reinterpret_cast<const double2*>(Ap);
    for (int64_t l = (int64_t)blockIdx.x * VEC_BLOCK + threadIdx.x; l < n2; l += stride) {
      double2 xv = x2[l], pv = p2[l], rv = r2[l], av = a2[l];
      xv.x = fma(alpha, pv.x, xv.x); xv.y = fma(alpha, pv.y, xv.y);
      rv.x = fma(-alpha, av.x, rv.x); rv.y = fma(-alpha, av.y, rv.y);
      x2[l] = xv; r2[l] = rv;
      acc = fma(rv.x, rv.x, acc); acc = fma(rv.y, rv.y, acc);
      if (invd) {
        const double2 dv = d2[l];
        acc_rz = fma(rv.x, rv.x * dv.x, acc_rz); acc_rz = fma(rv.y, rv.y * dv.y, acc_rz);
      }
    }
    if ((n & 1) && blockIdx.x == 0 && threadIdx.x == 0) {
      const int64_t l = n - 1;
      x[l] = fma(alpha, p[l], x[l]);
      const double rv = fma(-alpha, Ap[l], r[l]);
      r[l] = rv;
      acc = fma(rv, rv, acc);
      if (invd) acc_rz = fma(rv, rv * invd[l], acc_rz);
    }
  }
  acc = block_sum(acc);
  if (threadIdx.x == 0) rr_part[blockIdx.x] = acc;
  if (invd) {
    __syncthreads();
    acc_rz = block_sum(acc_rz);
    if (threadIdx.x == 0) rz_part[blockIdx.x] = acc_rz;
  }
  cooperative_groups::this_grid().sync();
  // ---- beta (identical in every CTA), p update + p.p
  double rn = 0.0, zn = 0.0;
  for (int b = threadIdx.x; b < (int)gridDim.x; b += VEC_BLOCK) rn += __ldcg(rr_part + b);
  rn = block_sum(rn);
  if (threadIdx.x == 0) s_b[1] = rn;
  if (invd) {
    __syncthreads();
    for (int b = threadIdx.x; b < (int)gridDim.x; b += VEC_BLOCK) zn += __ldcg(rz_part + b);
    zn = block_sum(zn);
    if (threadIdx.x == 0) s_b[2] = zn;
  }
  __syncthreads();
  const double rr_new = s_b[1];
  const double rho_new = invd ? s_b[2] : rr_new;
  const double beta = (rho != 0.0) ? rho_new / rho : 0.0;  // c15 guard
  double acc2 = 0.0;
  {
    double2* p2 = reinterpret_cast<double2*>(p);
    const double2* r2 = reinterpret_cast<const double2*>(r);
    double2* a2 = reinterpret_cast<double2*>(Ap);
    for (int64_t l = (int64_t)blockIdx.x * VEC_BLOCK + threadIdx.x; l < n2; l += stride) {
      double2 pv = p2[l], rv = __ldcg(r2 + l);
      if (invd) {  // z = M^-1 r
        const double2 dv = d2[l];
        rv.x *= dv.x; rv.y *= dv.y;
      }
      pv.x = fma(beta, pv.x, rv.x); pv.y = fma(beta, pv.y, rv.y);
      p2[l] = pv;
      a2[l] = make_double2(lam_init * pv.x, lam_init * pv.y);
      acc2 = fma(pv.x, pv.x, acc2); acc2 = fma(pv.y, pv.y, acc2);
    }
    if ((n & 1) && blockIdx.x == 0 && threadIdx.x == 0) {
      const int64_t l = n - 1;
      const double pv = fma(beta, p[l], __ldcg(r + l) * (invd ? invd[l] : 1.0));
      p[l] = pv; Ap[l] = lam_init * pv;
      acc2 = fma(pv, pv, acc2);
    }
  }
  acc2 = block_sum(acc2);
  if (threadIdx.x == 0) {
    pp_part[blockIdx.x] = acc2;  // every CTA read the old partials before the grid barrier
    if (blockIdx.x == 0) {
      s->pAp = pAp;
      s->rr = rr;
      if (hist) hist[s->it] = rr;
      s->rr_new = rr_new;
      s->rr_loc = rr_new;
      s->rz = rho_new;
      s->it += 1;
      if constexpr (COND) {
        if (ct.on) cond_test(ct, s, pAp, rr_new, s->it);
      }
    }
  }
}

template <int U, int MINB, bool COND>
__global__ void __launch_bounds__(VEC_BLOCK, MINB)
cg_update_fused(double* __restrict__ x, double* __restrict__ p, double* __restrict__ r, double* __restrict__ Ap,
                int64_t n, const double* __restrict__ e_part, int n_epart, double* pp_part, double lam_pp,
                double lam_init, double* rr_part, CgScalars* s, double* hist, const double* __restrict__ invd,
                double* rz_part, CondTest ct) {
  // U double2 per thread per batch: every load of a batch is issued before any use, and the
  // first batch is in flight while the CTA reduces the p.Ap partials.  When a thread's whole
  // share fits one batch, the p update reuses the registers (r_{j+1}, p_j, M^-1) -- no re-read.
  __shared__ double s_b[3];
  pdl_wait();
  const int64_t n2 = n >> 1;
  const int64_t stride = (int64_t)gridDim.x * VEC_BLOCK;
  const int64_t tid = (int64_t)blockIdx.x * VEC_BLOCK + threadIdx.x;
  const bool one = n2 <= (int64_t)U * stride;  // grid-uniform
  double2* x2 = reinterpret_cast<double2*>(x);
  double2* r2 = reinterpret_cast<double2*>(r);
  double2* p2 = reinterpret_cast<double2*>(p);
  double2* a2 = reinterpret_cast<double2*>(Ap);
  const double2* d2 = reinterpret_cast<const double2*>(invd);
  double2 xv[U], pv[U], rv[U], av[U], dv[U];
  auto load1 = [&](int64_t l0) {
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t l = l0 + u * stride;
      if (l < n2) {
        xv[u] = x2[l]; pv[u] = p2[l]; rv[u] = r2[l]; av[u] = a2[l];
        if (invd) dv[u] = d2[l];
      }
    }
  };
  if (tid < n2) load1(tid);
  // ---- p.Ap and alpha (identical in every CTA)
  double ev = 0.0, pv_ = 0.0;
  for (int b = threadIdx.x; b < n_epart; b += VEC_BLOCK) ev += e_part[b];
  for (int b = threadIdx.x; b < (int)gridDim.x; b += VEC_BLOCK) pv_ += pp_part[b];
  ev = block_sum(ev);
  __syncthreads();
  pv_ = block_sum(pv_);
  const double rr = s->rr_new;             // r_j.r_j
  const double rho = invd ? s->rz : rr;     // r_j.z_j (PCG) or r_j.r_j (CG)
  if (threadIdx.x == 0) s_b[0] = ev + lam_pp * pv_;
  __syncthreads();
  const double pAp = s_b[0];
  const double alpha = (pAp != 0.0) ? rho / pAp : 0.0;  // c15 guard
  // ---- x, r update + r.r (+ r.z)
  double acc = 0.0, acc_rz = 0.0;
  for (int64_t l0 = tid; l0 < n2;) {
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t l = l0 + u * stride;
      if (l < n2) {
        xv[u].x = fma(alpha, pv[u].x, xv[u].x); xv[u].y = fma(alpha, pv[u].y, xv[u].y);
        rv[u].x = fma(-alpha, av[u].x, rv[u].x); rv[u].y = fma(-alpha, av[u].y, rv[u].y);
        x2[l] = xv[u]; r2[l] = rv[u];
        acc = fma(rv[u].x, rv[u].x, acc); acc = fma(rv[u].y, rv[u].y, acc);
        if (invd) {
          acc_rz = fma(rv[u].x, rv[u].x * dv[u].x, acc_rz); acc_rz = fma(rv[u].y, rv[u].y * dv[u].y, acc_rz);
        }
      }
    }
    l0 += (int64_t)U * stride;
    if (l0 < n2) load1(l0);
  }
  if ((n & 1) && blockIdx.x == 0 && threadIdx.x == 0) {
    const int64_t l = n - 1;
    x[l] = fma(alpha, p[l], x[l]);
    const double rvl = fma(-alpha, Ap[l], r[l]);
    r[l] = rvl;
    acc = fma(rvl, rvl, acc);
    if (invd) acc_rz = fma(rvl, rvl * invd[l], acc_rz);
  }
  acc = block_sum(acc);
  if (threadIdx.x == 0) rr_part[blockIdx.x] = acc;
  if (invd) {
    __syncthreads();
    acc_rz = block_sum(acc_rz);
    if (threadIdx.x == 0) rz_part[blockIdx.x] = acc_rz;
  }
  cooperative_groups::this_grid().sync();
  // ---- beta (identical in every CTA), p update + p.p
  double rn = 0.0, zn = 0.0;
  for (int b = threadIdx.x; b < (int)gridDim.x; b += VEC_BLOCK) rn += __ldcg(rr_part + b);
  rn = block_sum(rn);
  if (threadIdx.x == 0) s_b[1] = rn;
  if (invd) {
    __syncthreads();
    for (int b = threadIdx.x; b < (int)gridDim.x; b += VEC_BLOCK) zn += __ldcg(rz_part + b);
    zn = block_sum(zn);
    if (threadIdx.x == 0) s_b[2] = zn;
  }
  __syncthreads();
  const double rr_new = s_b[1];
  const double rho_new = invd ? s_b[2] : rr_new;
  const double beta = (rho != 0.0) ? rho_new / rho : 0.0;  // c15 guard
  double acc2 = 0.0;
  auto pupd = [&](int64_t l, double2 pvv, double2 rvv, double2 dvv) {
    if (invd) { rvv.x *= dvv.x; rvv.y *= dvv.y; }  // z = M^-1 r
    pvv.x = fma(beta, pvv.x, rvv.x); pvv.y = fma(beta, pvv.y, rvv.y);
    p2[l] = pvv;
    a2[l] = make_double2(lam_init * pvv.x, lam_init * pvv.y);
    acc2 = fma(pvv.x, pvv.x, acc2); acc2 = fma(pvv.y, pvv.y, acc2);
  };
  if (one) {  // this thread's r_{j+1}, p_j (and M^-1) are still in registers
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t l = tid + u * stride;
      if (l < n2) pupd(l, pv[u], rv[u], invd ? dv[u] : make_double2(0.0, 0.0));
    }
  } else {
    for (int64_t l0 = tid; l0 < n2; l0 += (int64_t)U * stride) {
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int64_t l = l0 + u * stride;
        if (l < n2) {
          pv[u] = p2[l]; rv[u] = __ldcg(r2 + l);
          if (invd) dv[u] = d2[l];
        }
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int64_t l = l0 + u * stride;
        if (l < n2) pupd(l, pv[u], rv[u], invd ? dv[u] : make_double2(0.0, 0.0));
      }
    }
  }
  if ((n & 1) && blockIdx.x == 0 && threadIdx.x == 0) {
    const int64_t l = n - 1;
    const double pvl = fma(beta, p[l], __ldcg(r + l) * (invd ? invd[l] : 1.0));
    p[l] = pvl; Ap[l] = lam_init * pvl;
    acc2 = fma(pvl, pvl, acc2);
  }
  acc2 = block_sum(acc2);
  if (threadIdx.x == 0) {
    pp_part[blockIdx.x] = acc2;  // every CTA read the old partials before the grid barrier
    if (blockIdx.x == 0) {
      s->pAp = pAp;
      s->rr = rr;
      if (hist) hist[s->it] = rr;
      s->rr_new = rr_new;
      s->rr_loc = rr_new;
      s->rz = rho_new;
      s->it += 1;
      if constexpr (COND) {
        if (ct.on) cond_test(ct, s, pAp, rr_new, s->it);
      }
    }
  }
}

// Split form used with P > 1: r -= alpha Ap with r.r first, so the r.r allreduce can
// run on the communication stream while x += alpha p executes ("hidden behind the AXPY").
__global__ void __launch_bounds__(VEC_BLOCK)
cg_update_r(double* __restrict__ r, const double* __restrict__ Ap, int64_t n, double* partials, CgScalars* s) {
  if (s->flags & 2) return;  // tolerance-mode solve already finished (the rest of the chunk is idle)
  const double pAp = s->pAp;
  const double alpha = (pAp != 0.0) ? s->rr / pAp : 0.0;  // c15 guard
  double acc = 0.0;
  const int64_t n2 = n >> 1;
  double2* r2 = reinterpret_cast<double2*>(r);
  const double2* a2 = reinterpret_cast<const double2*>(Ap);
  for (int64_t l = (int64_t)blockIdx.x * VEC_BLOCK + threadIdx.x; l < n2; l += (int64_t)gridDim.x * VEC_BLOCK) {
    double2 rv = r2[l], av = a2[l];
    rv.x = fma(-alpha, av.x, rv.x); rv.y = fma(-alpha, av.y, rv.y);
    r2[l] = rv;
    acc = fma(rv.x, rv.x, acc); acc = fma(rv.y, rv.y, acc);
  }
  if ((n & 1) && blockIdx.x == 0 && threadIdx.x == 0) {
    const int64_t l = n - 1;
    double rv = fma(-alpha, Ap[l], r[l]);
    r[l] = rv;
    acc = fma(rv, rv, acc);
  }
  double tot;
  if (finish_reduction(acc, partials, &s->ticket, &tot)) s->rr_loc = tot;
}

__global__ void __launch_bounds__(VEC_BLOCK)
cg_update_x(double* __restrict__ x, const double* __restrict__ p, int64_t n, const CgScalars* s) {
  if (s->flags & 2) return;
  const double pAp = s->pAp;
  const double alpha = (pAp != 0.0) ? s->rr / pAp : 0.0;
  const int64_t n2 = n >> 1;
  double2* x2 = reinterpret_cast<double2*>(x);
  const double2* p2 = reinterpret_cast<const double2*>(p);
  for (int64_t l = (int64_t)blockIdx.x * VEC_BLOCK + threadIdx.x; l < n2; l += (int64_t)gridDim.x * VEC_BLOCK) {
    double2 xv = x2[l], pv = p2[l];
    xv.x = fma(alpha, pv.x, xv.x); xv.y = fma(alpha, pv.y, xv.y);
    x2[l] = xv;
  }
  if ((n & 1) && blockIdx.x == 0 && threadIdx.x == 0) x[n - 1] = fma(alpha, p[n - 1], x[n - 1]);
}

// beta = rr_loc / rr;  p = r + beta p;  Ap = lam_init p (assembly init of the next apply);
// partial p.p -> pp (lambda term of the next fused p.Ap); rr_new = rr_loc; j += 1.
// Tolerance mode with P > 1 (eps >= 0; the solve runs in chunks of iterations without host round
// trips): the last CTA also takes Alg. 1's loop test (while r.r > eps), the iteration cap and
// the breakdown check (p.Ap <= 0 or non-finite, R4) and sets flags bit 1, after which every
// iteration kernel of the chunk returns at once (bit 0 as well on breakdown, j not advanced).
__global__ void __launch_bounds__(VEC_BLOCK)
cg_update_p(double* __restrict__ p, const double* __restrict__ r, double* __restrict__ Ap,
            int64_t n, double lam_init, double* partials, CgScalars* s, double eps, int32_t max_iters) {
  if (s->flags & 2) return;
  const double rr = s->rr, rrn = s->rr_loc;
  const double beta = (rr != 0.0) ? rrn / rr : 0.0;  // c15 guard
  double acc = 0.0;
  const int64_t n2 = n >> 1;
  double2* p2 = reinterpret_cast<double2*>(p);
  const double2* r2 = reinterpret_cast<const double2*>(r);
  double2* a2 = reinterpret_cast<double2*>(Ap);
  for (int64_t l = (int64_t)blockIdx.x * VEC_BLOCK + threadIdx.x; l < n2; l += (int64_t)gridDim.x * VEC_BLOCK) {
    double2 pv = p2[l], rv = r2[l];
    pv.x = fma(beta, pv.x, rv.x); pv.y = fma(beta, pv.y, rv.y);
    p2[l] = pv;
    a2[l] = make_double2(lam_init * pv.x, lam_init * pv.y);
    acc = fma(pv.x, pv.x, acc); acc = fma(pv.y, pv.y, acc);
  }
  if ((n & 1) && blockIdx.x == 0 && threadIdx.x == 0) {
    const int64_t l = n - 1;
    double pv = fma(beta, p[l], r[l]);
    p[l] = pv; Ap[l] = lam_init * pv;
    acc = fma(pv, pv, acc);
  }
  double tot;
  if (finish_reduction(acc, partials, &s->ticket, &tot)) {
    s->pp = tot;
    s->rr_new = rrn;
    if (eps >= 0.0) {
      const double pAp = s->pAp;
      if (!(pAp > 0.0) || !isfinite(pAp) || !isfinite(rrn)) {
        s->flags |= 3;
        return;
      }
    }
    s->it += 1;
    if (eps >= 0.0 && (!(rrn > eps) || s->it >= max_iters)) s->flags |= 2;
  }
}

// Device-side loop test of the tolerance-mode graph (Alg. 1 line 6: while r.r > eps), with
// the iteration cap and the breakdown check (p.Ap <= 0 or non-finite) folded in; sets the
// WHILE node's condition so the solve runs without host round trips.
__global__ void cg_continue(cudaGraphConditionalHandle h, CgScalars* s, double eps, int32_t max_iters, int first) {
  bool go = s->rr_new > eps && s->it < max_iters;
  if (!first) {
    const bool brk = !(s->pAp > 0.0) || !isfinite(s->pAp) || !isfinite(s->rr_new);
    if (brk) { s->flags |= 1; go = false; }
  } else {
    s->flags = 0;
  }
  cudaGraphSetConditional(h, go ? 1u : 0u);
}

// Deterministic assembly (P:219's gather Z^T through a CSR, K5): y[g] = lam0 x[g] +
// sum_{t in row g} yL[slot[t]], rows in ascending (e, n) slot order -- a fixed summation
// order, so the result is bitwise reproducible (the fused variant uses fp64 RED instead).
__global__ void __launch_bounds__(VEC_BLOCK)
csr_gather_kernel(const int32_t* __restrict__ row_ptr, const int32_t* __restrict__ slots,
                  const double* __restrict__ yL, const double* __restrict__ x, double lam0, double* __restrict__ y,
                  int64_t n) {
  for (int64_t g = (int64_t)blockIdx.x * VEC_BLOCK + threadIdx.x; g < n; g += (int64_t)gridDim.x * VEC_BLOCK) {
    double acc = lam0 * x[g];
    const int32_t t1 = row_ptr[g + 1];
    for (int32_t t = row_ptr[g]; t < t1; ++t) acc += yL[slots[t]];
    y[g] = acc;
  }
}

// ---- NekBone's scattered storage: vectors of length N_L
// (x_L = Z x_G), the operator (Z Z^T S_L + lambda I) x_L with a combined gather-scatter, and
// inner products weighted by the inverse counting vector W.

// w_L = Z Z^T yL + lambda p_L: one thread per global DOF sums its slots (CSR, ascending (e,n))
// and writes the sum to every slot.
__global__ void __launch_bounds__(VEC_BLOCK)
gs_scatter_kernel(const int32_t* __restrict__ row_ptr, const int32_t* __restrict__ slots,
                  const double* __restrict__ yL, const double* __restrict__ pL, double lam, double* __restrict__ wL,
                  int64_t n) {
  for (int64_t g = (int64_t)blockIdx.x * VEC_BLOCK + threadIdx.x; g < n; g += (int64_t)gridDim.x * VEC_BLOCK) {
    const int32_t t0 = row_ptr[g], t1 = row_ptr[g + 1];
    double acc = 0.0;
    for (int32_t t = t0; t < t1; ++t) acc += yL[slots[t]];
    for (int32_t t = t0; t < t1; ++t) {
      const int32_t sl = slots[t];
      wL[sl] = fma(lam, pL[sl], acc);
    }
  }
}

// W-weighted dot sum_s W_s a_s b_s -> *out (allreduce-free, P = 1)
__global__ void __launch_bounds__(VEC_BLOCK)
wdot_kernel(const double* __restrict__ W, const double* __restrict__ a, const double* __restrict__ b, int64_t n,
            double* partials, uint32_t* ticket, double* out) {
  double acc = 0.0;
  for (int64_t l = (int64_t)blockIdx.x * VEC_BLOCK + threadIdx.x; l < n; l += (int64_t)gridDim.x * VEC_BLOCK)
    acc = fma(W[l] * a[l], b[l], acc);
  double tot;
  if (finish_reduction(acc, partials, ticket, &tot)) *out = tot;
}

// alpha = rr / pAp; x += alpha p; r -= alpha w; W-weighted r.r -> rr_new (scattered CG)
__global__ void __launch_bounds__(VEC_BLOCK)
scat_update_xr(double* __restrict__ x, const double* __restrict__ p, double* __restrict__ r,
               const double* __restrict__ w, const double* __restrict__ W, int64_t n, double* partials, CgScalars* s,
               double* hist) {
  const double rr = s->rr_new;
  const double pAp = s->pAp;
  const double alpha = (pAp != 0.0) ? rr / pAp : 0.0;
  double acc = 0.0;
  for (int64_t l = (int64_t)blockIdx.x * VEC_BLOCK + threadIdx.x; l < n; l += (int64_t)gridDim.x * VEC_BLOCK) {
    x[l] = fma(alpha, p[l], x[l]);
    const double rv = fma(-alpha, w[l], r[l]);
    r[l] = rv;
    acc = fma(W[l] * rv, rv, acc);
  }
  double tot;
  if (finish_reduction(acc, partials, &s->ticket, &tot)) {
    s->rr = rr;
    if (hist) hist[s->it] = rr;
    s->rr_new = tot;
  }
}

// beta = rr_new / rr; p = r + beta p (scattered CG)
__global__ void __launch_bounds__(VEC_BLOCK)
scat_update_p(double* __restrict__ p, const double* __restrict__ r, int64_t n, CgScalars* s) {
  const double rr = s->rr;
  const double beta = (rr != 0.0) ? s->rr_new / rr : 0.0;
  for (int64_t l = (int64_t)blockIdx.x * VEC_BLOCK + threadIdx.x; l < n; l += (int64_t)gridDim.x * VEC_BLOCK)
    p[l] = fma(beta, p[l], r[l]);
  if (blockIdx.x == 0 && threadIdx.x == 0) s->it += 1;
}

// x_L = Z x_G (scatter) and x_G = one slot of each DOF (gather back of a scattered vector)
__global__ void __launch_bounds__(VEC_BLOCK)
scatter_kernel(const int32_t* __restrict__ idx, const double* __restrict__ xg, double* __restrict__ xl, int64_t nl) {
  for (int64_t s = (int64_t)blockIdx.x * VEC_BLOCK + threadIdx.x; s < nl; s += (int64_t)gridDim.x * VEC_BLOCK)
    xl[s] = xg[idx[s]];
}
__global__ void __launch_bounds__(VEC_BLOCK)
pick_kernel(const int32_t* __restrict__ row_ptr, const int32_t* __restrict__ slots, const double* __restrict__ xl,
            double* __restrict__ xg, int64_t n) {
  for (int64_t g = (int64_t)blockIdx.x * VEC_BLOCK + threadIdx.x; g < n; g += (int64_t)gridDim.x * VEC_BLOCK)
    xg[g] = xl[slots[row_ptr[g]]];
}

// Jacobi preconditioner (NekBone's "simple diagonal preconditioning",
// P:140): diag(A)_g = sum over the slots of g of (S_L^e)_nn (+ lambda B_n in mass mode 1);
// (S_L^e)_nn = sum_m D[m][i]^2 Grr(m,j,k) + D[m][j]^2 Gss(i,m,k) + D[m][k]^2 Gtt(i,j,m)
//            + 2 D[i][i] D[j][j] Grs + 2 D[i][i] D[k][k] Grt + 2 D[j][j] D[k][k] Gst  (node n).
// One thread per slot, fp64 RED into diag (setup only).
__global__ void jacobi_diag_kernel(const double* __restrict__ G, const int32_t* __restrict__ idx,
                                   const double* __restrict__ B, int64_t E, int N, double lam, double* diag) {
  const int NP = N + 1, NP2 = NP * NP, NP3 = NP2 * NP;
  const double* D = c_D[N];
  for (int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; s < E * NP3; s += (int64_t)gridDim.x * blockDim.x) {
    const int64_t e = s / NP3;
    const int n = (int)(s - e * NP3);
    const int k = n / NP2, c = n - k * NP2, i = c % NP, j = c / NP;
    const double* Ge = G + e * 6 * NP3;
    auto g = [&](int f, int ii, int jj, int kk) { return Ge[g_off(g_pairs(N), NP2, kk, f, jj * NP + ii)]; };
    double d = 0.0;
    for (int m = 0; m < NP; ++m) {
      d += D[m * NP + i] * D[m * NP + i] * g(0, m, j, k);
      d += D[m * NP + j] * D[m * NP + j] * g(3, i, m, k);
      d += D[m * NP + k] * D[m * NP + k] * g(5, i, j, m);
    }
    const double di = D[i * NP + i], dj = D[j * NP + j], dk = D[k * NP + k];
    d += 2.0 * (di * dj * g(1, i, j, k) + di * dk * g(2, i, j, k) + dj * dk * g(4, i, j, k));
    if (B) d += lam * B[s];
    atomicAdd(diag + idx[s], d);
  }
}

// invd = 1 / (diag + shift)   (shift = lambda in mass mode 0: Z^T lambda W Z = lambda I)
__global__ void invert_kernel(double* __restrict__ d, int64_t n, double shift) {
  for (int64_t l = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; l < n; l += (int64_t)gridDim.x * blockDim.x)
    d[l] = 1.0 / (d[l] + shift);
}

// generic dot a.b -> *out (used by hb_dot)
__global__ void __launch_bounds__(VEC_BLOCK)
vec_dot(const double* __restrict__ a, const double* __restrict__ b, int64_t n, double* partials,
        uint32_t* ticket, double* out) {
  double acc = 0.0;
  for (int64_t l = (int64_t)blockIdx.x * VEC_BLOCK + threadIdx.x; l < n; l += (int64_t)gridDim.x * VEC_BLOCK)
    acc = fma(a[l], b[l], acc);
  double tot;
  if (finish_reduction(acc, partials, ticket, &tot)) *out = tot;
}

// y = s * x
__global__ void __launch_bounds__(VEC_BLOCK)
vec_scale(const double* __restrict__ x, double* __restrict__ y, int64_t n, double s) {
  for (int64_t l = (int64_t)blockIdx.x * VEC_BLOCK + threadIdx.x; l < n; l += (int64_t)gridDim.x * VEC_BLOCK)
    y[l] = s * x[l];
}

// forcing b[l] = 2 (splitmix64(gid ^ seed) >> 11) 2^-53 - 1 (reading c12)
__device__ __forceinline__ uint64_t d_splitmix64(uint64_t z) {
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

__global__ void __launch_bounds__(VEC_BLOCK)
forcing_kernel(double* __restrict__ b, const int64_t* __restrict__ gids, int64_t n, uint64_t seed) {
  for (int64_t l = (int64_t)blockIdx.x * VEC_BLOCK + threadIdx.x; l < n; l += (int64_t)gridDim.x * VEC_BLOCK) {
    uint64_t g = gids ? (uint64_t)gids[l] : (uint64_t)l;
    uint64_t h = d_splitmix64(g ^ seed);
    b[l] = 2.0 * ((double)(h >> 11) * 0x1.0p-53) - 1.0;
  }
}

// 8:1 streaming kernel: each thread reads 8 fp64 and writes 1
__global__ void __launch_bounds__(VEC_BLOCK)
stream8to1(const double* __restrict__ in, double* __restrict__ out, int64_t n) {
  for (int64_t l = (int64_t)blockIdx.x * VEC_BLOCK + threadIdx.x; l < n; l += (int64_t)gridDim.x * VEC_BLOCK) {
    double s = 0.0;
#pragma unroll
    for (int k = 0; k < 8; ++k) s += __ldcs(in + (int64_t)k * n + l);
    __stcs(out + l, s);
  }
}

// halo pack: buf[t] = x[loc[t]]
__global__ void __launch_bounds__(VEC_BLOCK)
pack_kernel(const double* __restrict__ x, const int32_t* __restrict__ loc, double* __restrict__ buf, int64_t n) {
  for (int64_t t = (int64_t)blockIdx.x * VEC_BLOCK + threadIdx.x; t < n; t += (int64_t)gridDim.x * VEC_BLOCK)
    buf[t] = x[loc[t]];
}

// assembly unpack: y[loc[t]] += buf[t]  (entries of loc are distinct within one call)
__global__ void __launch_bounds__(VEC_BLOCK)
unpack_add_kernel(double* __restrict__ y, const int32_t* __restrict__ loc, const double* __restrict__ buf, int64_t n) {
  for (int64_t t = (int64_t)blockIdx.x * VEC_BLOCK + threadIdx.x; t < n; t += (int64_t)gridDim.x * VEC_BLOCK)
    atomicAdd(y + loc[t], buf[t]);
}

// IPC allreduce (op.cu ipc_allreduce): lane q stores this rank's value into rank q's mailbox
// slot vals[q][slot*P + me] (peer memory), then -- after a system-scope fence -- raises this
// rank's flag in rank q's mailbox to seq.  vals_tab / flag_tab: per-rank base pointers
// (peer-mapped, own entry local); P <= 32.
__global__ void ipc_push_kernel(const double* __restrict__ v, double* const* __restrict__ vals_tab,
                                uint32_t* const* __restrict__ flag_tab, int P, int me, int slot, uint32_t seq) {
  const int q = threadIdx.x;
  if (q >= P) return;
  vals_tab[q][slot * P + me] = *v;
  __threadfence_system();
  if (q != me) *(volatile uint32_t*)(flag_tab[q] + me) = seq;
}

// sum of the P slot values in rank order (identical on every rank: deterministic allreduce)
__global__ void ipc_sum_kernel(const double* vals, int P, double* out) {
  double s = 0.0;
  for (int q = 0; q < P; ++q) s += ((const volatile double*)vals)[q];
  *out = s;
}

}  // namespace hbk
