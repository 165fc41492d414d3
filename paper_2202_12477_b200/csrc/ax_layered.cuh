// Fused screened-Poisson operator kernel, "layered" variant (all N).
//
//   Ap[g] (+)= sum_{(e,n): idx[e][n] = g} ( S_L^e u_e + lambda M_e u_e )[n],  u_e[n] = x[idx[e][n]]
//
// P:94-99   S_L^e = bold-D^T G^e bold-D, bold-D = [D(x)I(x)I; I(x)D(x)I; I(x)I(x)D]
// P:100-108 six geometric factors per node
// P:154     one kernel for y_L = (S_L + lambda W) Z x_G; here Z^T is fused as well
//           (scatter-add into assembled storage), see DESIGN.md "Operator kernel".
//
// Thread mapping (the paper's 2-D "layered" structure): one thread per (i, j)
// column of an element, EPB elements per CTA.  Each thread keeps its k-column of u in
// registers, so the t-direction contraction is register-only with D from constant memory;
// the r/s contractions read the current k-layer from shared memory with D rows in
// registers.  Element-interior nodes (0<i,j,k<N) belong to exactly one element, so they
// are written with a plain store (their W = 1); boundary nodes use fp64 RED into an
// output pre-initialised to lambda*x by the CG p-update (Z^T W Z = I, reading c1).
#pragma once
#include <cstdint>

namespace hbk {

__constant__ double c_D[16][256];  // c_D[N][i*(N+1)+j] = D_ij for N = 1..15

struct AxArgs {
  const int32_t* __restrict__ idx;  // [E][NP3] local index into [owned | halo]
  const double* __restrict__ G;     // [E][NP][6][NP2] slab-major
  const double* __restrict__ B;     // [E][NP3] (mass mode 1) or null
  const double* __restrict__ x;     // owned values
  const double* __restrict__ xh;    // halo values (HALO)
  double* y;                        // owned output (pre-initialised)
  double* yh;                       // halo output accumulator (HALO)
  int64_t e_begin, e_end;           // element range of this launch
  int32_t n_owned;
  double lam;
};

template <int N>
struct AxShape {
  static constexpr int NP = N + 1;
  static constexpr int NP2 = NP * NP;
  static constexpr int NP3 = NP2 * NP;
  static constexpr int EPB = (128 / NP2) > 0 ? (128 / NP2) : 1;
  static constexpr int BLOCK = EPB * NP2;
  // D rows in registers for small N; padded shared-memory copies for N >= 9 (register budget)
  static constexpr bool DREG = (N <= 8);
  static constexpr int LDD = NP + 1;
  static constexpr size_t SMEM = sizeof(double) * (3 * EPB * NP3 + (DREG ? 0 : NP * LDD));
};

template <bool HALO>
__device__ __forceinline__ double load_x(const AxArgs& a, int32_t g) {
  if (HALO && g >= a.n_owned) return a.xh[g - a.n_owned];
  return __ldg(a.x + g);
}

template <bool HALO>
__device__ __forceinline__ void red_y(const AxArgs& a, int32_t g, double v) {
  if (HALO && g >= a.n_owned) atomicAdd(a.yh + (g - a.n_owned), v);
  else atomicAdd(a.y + g, v);
}

// L2 prefetch of a contiguous byte range by the bulk-copy engine (sm_90+): no registers,
// no shared memory; keeps HBM streaming while the SM works on earlier elements.
__device__ __forceinline__ void prefetch_l2_bulk(const void* p, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(bytes) : "memory");
}

// MINB: minimum resident CTAs per SM requested from ptxas (register cap); PF: L2 prefetch
// distance in grid-stride waves (0 = off).
template <int N, bool HALO, bool MASSB, int MINB = 1, int PF = 0>
__global__ void __launch_bounds__(AxShape<N>::BLOCK, MINB)
ax_layered(const AxArgs a) {
  using S = AxShape<N>;
  constexpr int NP = S::NP, NP2 = S::NP2, NP3 = S::NP3, EPB = S::EPB;
  extern __shared__ double smem[];
  double(*s_u)[NP3] = reinterpret_cast<double(*)[NP3]>(smem);
  double(*s_r)[NP3] = reinterpret_cast<double(*)[NP3]>(smem + EPB * NP3);
  double(*s_s)[NP3] = reinterpret_cast<double(*)[NP3]>(smem + 2 * EPB * NP3);
  double* s_D = smem + 3 * EPB * NP3;  // [NP][LDD] (only when !DREG)
  constexpr int LDD = S::LDD;

  const int t = threadIdx.x;
  const int le = t / NP2;
  const int c = t - le * NP2;
  const int i = c % NP, j = c / NP;

  // D_ri = D[i][m], D_sj = D[j][m], DT_i = D[m][i], DT_j = D[m][j]
  double Dri[S::DREG ? NP : 1], Dsj[S::DREG ? NP : 1], DTi[S::DREG ? NP : 1], DTj[S::DREG ? NP : 1];
  if constexpr (S::DREG) {
#pragma unroll
    for (int m = 0; m < NP; ++m) {
      Dri[m] = c_D[N][i * NP + m];
      Dsj[m] = c_D[N][j * NP + m];
      DTi[m] = c_D[N][m * NP + i];
      DTj[m] = c_D[N][m * NP + j];
    }
  } else {
    for (int q = t; q < NP * NP; q += blockDim.x) s_D[(q / NP) * LDD + q % NP] = c_D[N][q];
    __syncthreads();
  }
#define HB_DRI(m) (S::DREG ? Dri[(m) < NP ? (m) : 0] : s_D[i * LDD + (m)])
#define HB_DSJ(m) (S::DREG ? Dsj[(m) < NP ? (m) : 0] : s_D[j * LDD + (m)])
#define HB_DTI(m) (S::DREG ? DTi[(m) < NP ? (m) : 0] : s_D[(m) * LDD + i])
#define HB_DTJ(m) (S::DREG ? DTj[(m) < NP ? (m) : 0] : s_D[(m) * LDD + j])
  const bool interior_ij = (i > 0 && i < N && j > 0 && j < N);

  if constexpr (PF > 0) {  // prime: the first PF waves
    if (t == 0)
      for (int w = 0; w < PF; ++w) {
        const int64_t nb = a.e_begin + ((int64_t)blockIdx.x + (int64_t)w * gridDim.x) * EPB;
        if (nb < a.e_end) {
          const int64_t ne = (a.e_end - nb) < EPB ? (a.e_end - nb) : EPB;
          prefetch_l2_bulk(a.G + nb * 6 * NP3, (uint32_t)(ne * 6 * NP3 * sizeof(double)));
          prefetch_l2_bulk(a.idx + nb * NP3, (uint32_t)((ne * NP3 * sizeof(int32_t) + 15) & ~15u));
        }
      }
  }
  for (int64_t base = a.e_begin + (int64_t)blockIdx.x * EPB; base < a.e_end; base += (int64_t)gridDim.x * EPB) {
    if constexpr (PF > 0) {
      if (t == 0) {
        const int64_t nb = base + (int64_t)PF * gridDim.x * EPB;
        if (nb < a.e_end) {
          const int64_t ne = (a.e_end - nb) < EPB ? (a.e_end - nb) : EPB;
          prefetch_l2_bulk(a.G + nb * 6 * NP3, (uint32_t)(ne * 6 * NP3 * sizeof(double)));
          prefetch_l2_bulk(a.idx + nb * NP3, (uint32_t)((ne * NP3 * sizeof(int32_t) + 15) & ~15u));
        }
      }
    }
    const int64_t e = base + le;
    const bool act = (e < a.e_end);
    int32_t gi[NP];
    double u[NP];
    // gather u_e = Z x (indirect read of x_G)
#pragma unroll
    for (int k = 0; k < NP; ++k) {
      gi[k] = act ? __ldg(a.idx + e * NP3 + k * NP2 + c) : 0;
      u[k] = act ? load_x<HALO>(a, gi[k]) : 0.0;
    }
#pragma unroll
    for (int k = 0; k < NP; ++k) s_u[le][k * NP2 + c] = u[k];
    // t-direction gradient in registers: ut[k] = sum_m D[k][m] u[m]
    double wt[NP];
#pragma unroll
    for (int k = 0; k < NP; ++k) {
      double acc = 0.0;
#pragma unroll
      for (int m = 0; m < NP; ++m) acc = fma(c_D[N][k * NP + m], u[m], acc);
      wt[k] = acc;
    }
    __syncthreads();
    // r/s gradients per layer, metric (15 flops/node), stash r/s fluxes in smem
    const double* Ge = a.G + e * (6 * NP3);
#pragma unroll
    for (int k = 0; k < NP; ++k) {
      double ur = 0.0, us = 0.0;
#pragma unroll
      for (int m = 0; m < NP; ++m) {
        ur = fma(HB_DRI(m), s_u[le][k * NP2 + j * NP + m], ur);
        us = fma(HB_DSJ(m), s_u[le][k * NP2 + m * NP + i], us);
      }
      double grr = 0, grs = 0, grt = 0, gss = 0, gst = 0, gtt = 0;
      if (act) {
        const double* g = Ge + k * 6 * NP2 + c;
        grr = __ldg(g); grs = __ldg(g + NP2); grt = __ldg(g + 2 * NP2);
        gss = __ldg(g + 3 * NP2); gst = __ldg(g + 4 * NP2); gtt = __ldg(g + 5 * NP2);
      }
      const double ut = wt[k];
      s_r[le][k * NP2 + c] = grr * ur + grs * us + grt * ut;
      s_s[le][k * NP2 + c] = grs * ur + gss * us + gst * ut;
      wt[k] = grt * ur + gst * us + gtt * ut;
    }
    __syncthreads();
    // divergence bold-D^T and assembly Z^T
#pragma unroll
    for (int k = 0; k < NP; ++k) {
      double out = 0.0;
#pragma unroll
      for (int m = 0; m < NP; ++m) {
        out = fma(HB_DTI(m), s_r[le][k * NP2 + j * NP + m], out);
        out = fma(HB_DTJ(m), s_s[le][k * NP2 + m * NP + i], out);
        out = fma(c_D[N][m * NP + k], wt[m], out);
      }
      if (act) {
        const double uk = s_u[le][k * NP2 + c];
        if (MASSB) out = fma(a.lam * __ldg(a.B + e * NP3 + k * NP2 + c), uk, out);
        if (interior_ij && k > 0 && k < N) {
          if (!MASSB) out = fma(a.lam, uk, out);  // W = 1 on element-interior nodes
          a.y[gi[k]] = out;                       // sole contribution: plain store
        } else {
          red_y<HALO>(a, gi[k], out);
        }
      }
    }
    __syncthreads();
  }
#undef HB_DRI
#undef HB_DSJ
#undef HB_DTI
#undef HB_DTJ
}

}  // namespace hbk
