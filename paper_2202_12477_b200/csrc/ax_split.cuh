// Fused screened-Poisson operator kernel, "split-line" variant (sm_100a).
//
//   Ap[g] (+)= sum_{(e,n): idx[e][n] = g} ( S_L^e u_e + lambda M_e u_e )[n],  u_e[n] = x[idx[e][n]]
//
// P:94-99   S_L^e = bold-D^T G^e bold-D;  P:100-108 six geometric factors (15 flops/node);
// P:154     one kernel for (S_L + lambda W) Z x_G, Z^T fused (scatter-add).
//
// Same arithmetic as ax_lines.cuh (even/odd folded 1-D contractions with warp-uniform D
// broadcasts, shared-memory transposes between the three line orientations), but each element
// is worked by 2 (N+1)^2 threads instead of (N+1)^2.  Thread (c, h), c = (i,j) column, h in {0,1}:
//   * t-direction: both threads of column c read the whole column and fold it; thread h forms
//     the outputs of its half of the row pairs (i, N-i) (and the middle row, h = 1, N+1 odd).
//     Its column nodes (ca, cb, k in rows(h)) are its own for the gather, the metric and the
//     assembly, so u, the index and the t-derivatives stay in its registers;
//   * r- and s-directions: thread (c, 0) owns the r-line (j,k) = c, thread (c, 1) the s-line
//     (i,k) = c, each contracted whole by one thread (streamed to shared memory).
// Twice the warps per element at about half the registers per thread: the large-N line kernel
// (one 256-thread CTA per SM at 255 registers for N = 15, 8 warps per SM) becomes latency-bound
// on its G loads and FMA chains; here every G load of P3 is issued by twice as many threads
// (half as many each, all hoisted), and no shared u is kept past the gather (4 barriers per
// element instead of 5).
//   P1  (c,h): gather u at its nodes (Z x) -> s_u, registers
//   P2  (c,h): t-half ut = (D u_col)[rows(h)] (registers);  r-line (h=0) -> s_r, s-line (h=1) -> s_s
//   P3  (c,h): metric at its nodes: gr -> s_r, gs -> s_s, gt -> s_u (in place)
//   P4  (c,h): t-half vt = (D^T gt_col)[rows(h)] (registers);  r-line D^T in place (h=0), s-line (h=1)
//   P5  (c,h): out = vt + vr + vs (+ lambda terms), element energy, assembly Z^T (store / RED)
#pragma once
#include <cstdint>
#include <type_traits>

#include "ax_lines.cuh"  // LinesShape (shared-memory layout, folded D table), dot_rows, ldG, energy_finish

namespace hbk {

template <int N, int EPBX = 0>
struct SplitShape {
  using L = LinesShape<N, EPBX>;
  static constexpr int NP = N + 1, NP2 = NP * NP, NP3 = NP2 * NP;
  static constexpr int H = L::H, ODD = L::ODD, HE = L::HE, HE2 = L::HE2, H2 = L::H2;
  static constexpr int EPB = EPBX > 0 ? EPBX : ((64 / NP2) > 0 ? (64 / NP2) : 1);
  static constexpr int TPE = 2 * NP2;  // threads per element
  static constexpr int BLOCK = EPB * TPE;
  static constexpr int SLAB = L::SLAB;
  static constexpr size_t SMEM = sizeof(double) * (3 * EPB * SLAB + L::CONST);
  // row pairs (p, N-p): p < HP0 to half 0, the rest (and the middle row, N+1 odd) to half 1
  static constexpr int HP0 = (H + 1) / 2;
  static constexpr int NPAIR0 = HP0, NPAIR1 = H - HP0;
  static constexpr int RH0 = 2 * NPAIR0, RH1 = 2 * NPAIR1 + ODD;
  static constexpr int RHM = RH0 > RH1 ? RH0 : RH1;
  // register target per N (resident CTAs requested from ptxas), capped by shared memory
  static constexpr int REGS_T[16] = {0, 64, 64, 64, 64, 64, 64, 64, 80, 80, 80, 96, 96, 128, 128, 128};
  static constexpr int REGS = REGS_T[N];
  static constexpr int MINB_REG0 = 65536 / (BLOCK * REGS);
  static constexpr int MINB_REG = MINB_REG0 < 1 ? 1 : (MINB_REG0 > 16 ? 16 : MINB_REG0);
  static constexpr int MINB_SMEM = (int)((227 * 1024) / (SMEM + 1024));
  static constexpr int MINB = MINB_REG < MINB_SMEM ? MINB_REG : (MINB_SMEM < 1 ? 1 : MINB_SMEM);
};

// Rows (t-direction k / output index) of half HH: q = 2 (p - P0) -> p, q = 2 (p - P0) + 1 -> N - p,
// q = RH - 1 -> the middle row (half 1, N+1 odd).
template <int N, int HH>
struct SplitHalf {
  using S = SplitShape<N>;
  static constexpr int P0 = HH == 0 ? 0 : S::HP0;
  static constexpr int NPAIR = HH == 0 ? S::NPAIR0 : S::NPAIR1;
  static constexpr bool MID = HH == 1 && S::ODD;
  static constexpr int RH = 2 * NPAIR + (MID ? 1 : 0);
  __device__ __forceinline__ static constexpr int row(int q) {
    return (MID && q == RH - 1) ? S::H : ((q & 1) ? N - (P0 + q / 2) : (P0 + q / 2));
  }
};

// Fold a line v[0..N] in place: v[m] <- e_m = v_m + v_{N-m}, v[N-m] <- o_m = v_m - v_{N-m}
// (m < H); the middle value (N+1 odd) is its own e.  e_m then lives at v[m], o_m at v[N-m].
template <int N>
__device__ __forceinline__ void fold_line(double (&v)[N + 1]) {
  constexpr int H = (N + 1) / 2;
#pragma unroll
  for (int m = 0; m < H; ++m) {
    const double a = v[m], b = v[N - m];
    v[m] = a + b;
    v[N - m] = a - b;
  }
}

// Row pair p of the folded operator on a folded line: y_p = so + se, y_{N-p} = so - se.
template <int N>
__device__ __forceinline__ void pair_rows(const double* __restrict__ sM, const double (&v)[N + 1], int p,
                                          double& yp, double& ymp) {
  using L = LinesShape<N>;
  constexpr int H = L::H, HE = L::HE, HE2 = L::HE2, H2 = L::H2;
  const double* Me = sM + p * HE2;
  const double* Mo = sM + H * HE2 + p * H2;
  double se = 0.0, so = 0.0;
#pragma unroll
  for (int m = 0; m + 1 < HE; m += 2) {
    const double2 c = *reinterpret_cast<const double2*>(Me + m);
    se = fma(c.x, v[m], se);
    se = fma(c.y, v[m + 1], se);
  }
  if constexpr (HE & 1) se = fma(Me[HE - 1], v[HE - 1], se);
#pragma unroll
  for (int m = 0; m + 1 < H; m += 2) {
    const double2 c = *reinterpret_cast<const double2*>(Mo + m);
    so = fma(c.x, v[N - m], so);
    so = fma(c.y, v[N - m - 1], so);
  }
  if constexpr (H & 1) so = fma(Mo[H - 1], v[N - (H - 1)], so);
  yp = so + se;
  ymp = so - se;
}

// middle row (N+1 odd): y_H = Mm . o
template <int N>
__device__ __forceinline__ double mid_row(const double* __restrict__ sM, const double (&v)[N + 1]) {
  using L = LinesShape<N>;
  constexpr int H = L::H, HE2 = L::HE2, H2 = L::H2;
  const double* Mm = sM + H * HE2 + H * H2;
  double s = 0.0;
#pragma unroll
  for (int m = 0; m + 1 < H; m += 2) {
    const double2 c = *reinterpret_cast<const double2*>(Mm + m);
    s = fma(c.x, v[N - m], s);
    s = fma(c.y, v[N - m - 1], s);
  }
  if constexpr (H & 1) s = fma(Mm[H - 1], v[N - (H - 1)], s);
  return s;
}

// Half HH of the t-contraction of one folded column: out[q] = (M col)[row(q)].
template <int N, int HH>
__device__ __forceinline__ void t_half(const double* __restrict__ sM, const double (&v)[N + 1],
                                       double (&out)[SplitShape<N>::RHM]) {
  using HS = SplitHalf<N, HH>;
#pragma unroll
  for (int q = 0; q < 2 * HS::NPAIR; q += 2) pair_rows<N>(sM, v, HS::P0 + q / 2, out[q], out[q + 1]);
  if constexpr (HS::MID) out[HS::RH - 1] = mid_row<N>(sM, v);
}

// Whole-line contraction, outputs streamed to sink(i, y_i) (one owner per line).
template <int N, class Sink>
__device__ __forceinline__ void full_line(const double* __restrict__ sM, const double (&v)[N + 1], Sink&& sink) {
  using L = LinesShape<N>;
  constexpr int H = L::H;
#pragma unroll
  for (int p = 0; p < H; ++p) {
    double a, b;
    pair_rows<N>(sM, v, p, a, b);
    sink(p, a);
    sink(N - p, b);
  }
  if constexpr (L::ODD) sink(H, mid_row<N>(sM, v));
}

template <int N, bool HALO, bool MASSB, int MINB = SplitShape<N>::MINB, int EPBX = 0,
          int PFL = LinesShape<N>::PFL_DEF, bool GCS = true>
__global__ void __launch_bounds__(SplitShape<N, EPBX>::BLOCK, MINB)
ax_split(const AxArgs a) {
  using S = SplitShape<N, EPBX>;
  using L = LinesShape<N, EPBX>;
  constexpr int NP = S::NP, NP2 = S::NP2, NP3 = S::NP3, EPB = S::EPB, SLAB = S::SLAB, RHM = S::RHM;
  extern __shared__ double smem[];
  const int t = threadIdx.x;
  const int le = t / S::TPE;
  const int r = t - le * S::TPE;
  const int h = r >= NP2 ? 1 : 0;
  const int c = r - h * NP2;
  const int ca = c % NP, cb = c / NP;  // (i,j) for the column, (j,k) r-line (h=0), (i,k) s-line (h=1)
  double* s_u = smem + (0 * EPB + le) * SLAB;
  double* s_r = smem + (1 * EPB + le) * SLAB;
  double* s_s = smem + (2 * EPB + le) * SLAB;
  double* s_D = smem + 3 * EPB * SLAB;  // folded D
  double* s_DT = s_D + L::MAT;          // folded D^T
  for (int q = t; q < L::CONST; q += S::BLOCK) s_D[q] = __ldg(&g_EO[N][q]);
  const bool interior_ij = (ca > 0 && ca < N && cb > 0 && cb < N);
  double en = 0.0;
  __syncthreads();

  for (int64_t base = a.e_begin + (int64_t)blockIdx.x * EPB; base < a.e_end; base += (int64_t)gridDim.x * EPB) {
    const int64_t e = base + le;
    const bool act = (e < a.e_end);
    if constexpr (PFL) {  // L2 prefetch of this element's G (consumed in P3) and the next element's index block
      if (act) {
        const char* gb = reinterpret_cast<const char*>(a.G + e * (6 * NP3));
        if constexpr (PFL == 2) {
          if (r == 0) prefetch_l2_bulk(gb, 48 * NP3);
        } else {
          for (int q = r; q < (6 * NP3 * 8) / 128; q += S::TPE) prefetch_l2_line(gb + q * 128);
        }
        const int64_t en_ = e + (int64_t)gridDim.x * EPB;
        if (en_ < a.e_end) {
          const char* ib = reinterpret_cast<const char*>(a.idx + en_ * NP3);
          for (int q = r; q < (NP3 * 4 + 127) / 128; q += S::TPE) prefetch_l2_line(ib + q * 128);
        }
      }
    }
    int32_t gi[RHM];
    double uu[RHM], tv[RHM];

    // ---- P1: gather this thread's column nodes (Z x)
    auto p1 = [&](auto hh) {
      constexpr int HH = decltype(hh)::value;
      using HS = SplitHalf<N, HH>;
#pragma unroll
      for (int q = 0; q < HS::RH; ++q) gi[q] = act ? __ldg(a.idx + e * NP3 + HS::row(q) * NP2 + c) : 0;
#pragma unroll
      for (int q = 0; q < HS::RH; ++q) {
        uu[q] = act ? load_x<HALO>(a, gi[q]) : 0.0;
        s_u[L::at(ca, cb, HS::row(q))] = uu[q];
      }
    };
    if (h == 0) p1(std::integral_constant<int, 0>{});
    else p1(std::integral_constant<int, 1>{});
    __syncthreads();

    // ---- P2: t-half (registers) and the r-line (h=0) / s-line (h=1) gradient
    {
      double v[NP];
#pragma unroll
      for (int m = 0; m < NP; ++m) v[m] = s_u[L::at(ca, cb, m)];
      fold_line<N>(v);
      if (h == 0) t_half<N, 0>(s_D, v, tv);
      else t_half<N, 1>(s_D, v, tv);
      if (h == 0) {
#pragma unroll
        for (int m = 0; m < NP; ++m) v[m] = s_u[L::at(m, ca, cb)];
        fold_line<N>(v);
        full_line<N>(s_D, v, [&](int i, double y) { s_r[L::at(i, ca, cb)] = y; });
      } else {
#pragma unroll
        for (int m = 0; m < NP; ++m) v[m] = s_u[L::at(ca, m, cb)];
        fold_line<N>(v);
        full_line<N>(s_D, v, [&](int j, double y) { s_s[L::at(ca, j, cb)] = y; });
      }
    }
    __syncthreads();

    // ---- P3: metric at this thread's nodes; gt replaces u in s_u
    auto p3 = [&](auto hh) {
      constexpr int HH = decltype(hh)::value;
      using HS = SplitHalf<N, HH>;
      const double* Ge = a.G + e * (6 * NP3);
#pragma unroll
      for (int q = 0; q < HS::RH; ++q) {
        const int k = HS::row(q);
        double grr = 0, grs = 0, grt = 0, gss = 0, gst = 0, gtt = 0;
        if (act) {  // G is read once per apply: streaming loads (ptxas hoists them as registers allow)
          if constexpr (g_pairs(N)) {
            const double2* g2 = reinterpret_cast<const double2*>(Ge + g_off(true, NP2, k, 0, c));
            const double2 p0 = ldG2<GCS>(g2), p1_ = ldG2<GCS>(g2 + NP2), p2 = ldG2<GCS>(g2 + 2 * NP2);
            grr = p0.x; grs = p0.y; grt = p1_.x; gss = p1_.y; gst = p2.x; gtt = p2.y;
          } else {
            const double* gp = Ge + g_off(false, NP2, k, 0, c);
            grr = ldG<GCS>(gp); grs = ldG<GCS>(gp + NP2); grt = ldG<GCS>(gp + 2 * NP2);
            gss = ldG<GCS>(gp + 3 * NP2); gst = ldG<GCS>(gp + 4 * NP2); gtt = ldG<GCS>(gp + 5 * NP2);
          }
        }
        const int o = L::at(ca, cb, k);
        const double ur = s_r[o], us = s_s[o], ut = tv[q];
        s_r[o] = grr * ur + grs * us + grt * ut;
        s_s[o] = grs * ur + gss * us + gst * ut;
        s_u[o] = grt * ur + gst * us + gtt * ut;
      }
    };
    if (h == 0) p3(std::integral_constant<int, 0>{});
    else p3(std::integral_constant<int, 1>{});
    __syncthreads();

    // ---- P4: transposed t-half (registers) and r-line (h=0) / s-line (h=1) in place
    {
      double v[NP];
#pragma unroll
      for (int m = 0; m < NP; ++m) v[m] = s_u[L::at(ca, cb, m)];
      fold_line<N>(v);
      if (h == 0) t_half<N, 0>(s_DT, v, tv);
      else t_half<N, 1>(s_DT, v, tv);
      if (h == 0) {
#pragma unroll
        for (int m = 0; m < NP; ++m) v[m] = s_r[L::at(m, ca, cb)];
        fold_line<N>(v);
        full_line<N>(s_DT, v, [&](int i, double y) { s_r[L::at(i, ca, cb)] = y; });
      } else {
#pragma unroll
        for (int m = 0; m < NP; ++m) v[m] = s_s[L::at(ca, m, cb)];
        fold_line<N>(v);
        full_line<N>(s_DT, v, [&](int j, double y) { s_s[L::at(ca, j, cb)] = y; });
      }
    }
    __syncthreads();

    // ---- P5: sum of the three directions, lambda terms, element energy, assembly Z^T
    auto p5 = [&](auto hh) {
      constexpr int HH = decltype(hh)::value;
      using HS = SplitHalf<N, HH>;
#pragma unroll
      for (int q = 0; q < HS::RH; ++q) {
        const int k = HS::row(q);
        const int o = L::at(ca, cb, k);
        double out = tv[q] + s_r[o] + s_s[o];
        const double uk = uu[q];
        en = fma(uk, out, en);
        if (MASSB) {
          const double lb = a.lam * __ldg(a.B + e * NP3 + k * NP2 + c) * uk;
          out += lb;
          en = fma(uk, lb, en);
        }
        if (interior_ij && k > 0 && k < N) {
          if (!MASSB) out = fma(a.lam, uk, out);  // W = 1 on element-interior nodes
          a.y[gi[q]] = out;                       // sole contribution: plain store
        } else {
          red_y<HALO>(a, gi[q], out);
        }
      }
    };
    if (act) {
      if (h == 0) p5(std::integral_constant<int, 0>{});
      else p5(std::integral_constant<int, 1>{});
    }
    // no barrier: the next P1 writes s_u, whose last readers (P4) passed the barrier above;
    // P5's s_r / s_s reads precede this thread's arrival at the next P1 barrier
  }
  if (a.cg) {
    __syncthreads();
    energy_finish<S::BLOCK>(en, a, smem);
  }
}

}  // namespace hbk
