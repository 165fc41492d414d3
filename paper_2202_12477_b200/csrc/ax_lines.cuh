// Fused screened-Poisson operator kernel, "line-owner" variant (sm_100a, all N).
//
//   Ap[g] (+)= sum_{(e,n): idx[e][n] = g} ( S_L^e u_e + lambda M_e u_e )[n],  u_e[n] = x[idx[e][n]]
//
// P:94-99   S_L^e = bold-D^T G^e bold-D, bold-D = [D(x)I(x)I; I(x)D(x)I; I(x)I(x)D]
// P:100-108 six geometric factors per node (15 flops/node)
// P:154     one kernel for (S_L + lambda W) Z x_G, here with Z^T fused (scatter-add)
//
// Every 1-D contraction is done by a thread that owns a whole line of N+1 values in
// registers, so all lanes of a warp use the same entry of D at the same time: D is read from
// shared memory with warp-uniform (broadcast) loads.  The GLL derivative matrix is
// centro-antisymmetric, D[N-i][N-m] = -D[i][m] (so is D^T), which the contraction exploits
// (even/odd folding): with e_m = u_m + u_{N-m}, o_m = u_m - u_{N-m},
//   y_i = sum_m Mo[i][m] o_m + sum_m Me[i][m] e_m,  y_{N-i} = sum_m Mo o - sum_m Me e,
//   Me[i][m] = (D[i][m] + D[i][N-m]) / 2,  Mo[i][m] = (D[i][m] - D[i][N-m]) / 2,
// which halves the multiply-adds of the 12(N+1)^4 term (the FOM still counts P:110's flops).
// Shared memory transposes between the three line orientations:
//   P1  column owner (i,j): gather u[k] = x[idx] -> s_u; ut = D u (registers)
//   P2  row owner (j,k): ur = D u_row -> s_r  and  (i,k) owner: us = D u_col -> s_s
//   P3  column owner (i,j): (gr,gs,gt) = G (ur,us,ut) -> s_r, s_s in place, gt in registers
//   P4  row owner: vr = D^T gr in place;  (i,k) owner: vs = D^T gs in place
//   P5  column owner: out[k] = (D^T gt)[k] + vr + vs (+ lambda terms) -> store / RED
// Padded layout s[k][j][i] with row pitch P1 and layer pitch P2 (offline bank-conflict
// search) keeps all three orientations (nearly) conflict free.  G and idx of the element
// group PF grid-waves ahead are prefetched into L2 by the bulk-copy engine, so HBM keeps
// streaming while the SM computes.  Element-interior nodes (0<i,j,k<N) have one contributing
// slot and W = 1: plain store; all other nodes use fp64 RED into an output pre-initialised
// to lambda*x (reading R2).
#pragma once
#include <cstdint>
#include <type_traits>

#include "common.cuh"  // AxArgs, c_D, prefetch_l2_bulk, load_x / red_y

namespace hbk {

template <int N, int EPBX = 0>
struct LinesShape {
  static constexpr int NP = N + 1;
  static constexpr int NP2 = NP * NP;
  static constexpr int NP3 = NP2 * NP;
  // ~64 threads per CTA (one element from N = 7 up): fine-grained CTAs balance best; N = 5
  // measured best with ~128 (profiles/r1_tune.jsonl)
  static constexpr int EPB_DEF = N == 5 ? 128 / NP2 : ((64 / NP2) > 0 ? (64 / NP2) : 1);
  static constexpr int EPB = EPBX > 0 ? EPBX : EPB_DEF;
  // ALN (the N = 6 default; EPBX = 1 selects the blocked mapping): each 7-thread row of columns /
  // lines occupies 8 lanes (ca = t & 7, lane 7 idle), so the 56 threads still fill two warps
  // and every half-warp holds exactly two rows; with row pitch 7 and the rows of layer k
  // rotated by k (see at()) all three orientations are conflict free (model 616 -> 448 shared
  // wavefronts per element, scripts/smem_conflicts.py).  Inside the CG at the C3 box: 0.70 ->
  // 0.76 of peak with 80 registers (12 CTAs per SM; profiles/r2/aln/).  The same alignment at
  // N = 9-14 (rows of 10-15 columns on 16-lane boundaries, pitch 17) and rotated rows at N = 3
  // measured slower (-3..-40%): extra warps or spills outweigh the conflicts they remove
  static constexpr bool ALN = (EPBX == -1 || EPBX == 0) && N == 6;
  static constexpr int RW = 8;
  static constexpr int BLOCK = ALN ? NP * RW : EPB * NP2;
  // Shared-memory layout of one element buffer: (i,j,k) -> doubles.  NP = 8 and NP = 16 use an
  // XOR swizzle that makes all three line orientations conflict free; other N use row / layer
  // padding from an offline bank-conflict search.
  // Element slabs may be odd (the D copy after them is realigned).  N = 2, 4: odd slabs from the
  // conflict model (scripts/smem_conflicts.py, wavefronts per CTA: N = 2 360 -> 276, N = 4
  // 440 -> 400; measured +5% / +3% inside the CG, profiles/r2/pad/)
  static constexpr int PAD[16][3] = {{0, 0, 0}, {2, 5, 12}, {3, 18, 57}, {4, 19, 76}, {5, 25, 137}, {9, 54, 324},
                                     {7, 52, 370}, {8, 72, 576}, {9, 81, 730}, {10, 101, 1010}, {11, 121, 1332},
                                     {13, 156, 1872}, {13, 169, 2198}, {17, 238, 3332}, {15, 225, 3376}, {16, 256, 4096}};
  static constexpr int P1 = ALN ? 7 : PAD[N][0];
  static constexpr int P2 = ALN ? 55 : PAD[N][1];
  static constexpr int SLAB = ALN ? NP * P2 : PAD[N][2];  // doubles per element per buffer
  // the folded D copy in shared memory starts 16-byte aligned (pair loads)
  static constexpr int DOFF0 = 3 * EPB * SLAB;
  static constexpr int DOFF = DOFF0 + (DOFF0 & 1);
  __device__ __forceinline__ static int at(int i, int j, int k) {
    if constexpr (N == 7) return k * 72 + j * 8 + (i ^ (((j >> 1) + 4 * (k & 1)) & 7));
    else if constexpr (N == 15) return k * 256 + j * 16 + (i ^ j);
    else if constexpr (ALN) {
      const int v = i + k;
      return k * 55 + j * 7 + (v >= 7 ? v - 7 : v);  // rows of layer k rotated by k
    }
    else return k * P2 + j * P1 + i;
  }
  // even/odd folded operator: H = (N+1)/2 row pairs, HE = H (+1 middle column if N+1 odd);
  // rows padded to even length so pairs load as one 16-byte broadcast
  static constexpr int H = NP / 2, ODD = NP & 1, HE = H + ODD;
  static constexpr int HE2 = HE + (HE & 1), H2 = H + (H & 1);
  static constexpr int MAT = H * HE2 + H * H2 + H2;  // Me, Mo, middle row
  static constexpr int CONST = 2 * MAT;               // D and D^T (host-built, g_EO[N])
  static_assert(CONST <= EO_MAX, "folded D table");
  static_assert(CONST == eo_const(N), "packed constant-memory D table");
  static constexpr size_t SMEM = sizeof(double) * (DOFF + CONST);
  // Line contractions: 0 = two lines (P2, P4) into output arrays; 1 = one line at a time, every
  // output streamed to shared memory / the assembly as it is formed; 2 = two lines streamed (D
  // read once per two lines, no output arrays).  GIR: the index column is re-read in P5 instead of
  // held in registers from P1.  Streaming frees the registers for two CTAs per SM at N = 11, 12:
  // N = 11 0.78 -> 0.83 isolated, 0.65 -> 0.74 inside the CG (2 lines, index re-read, 128
  // registers), N = 12 0.69 -> 0.76 / 0.65 -> 0.70 (2 lines, 168 registers).  N = 13 gains in
  // isolation (0.62 -> 0.69) but loses inside the CG (0.61 -> 0.55) and keeps one uncapped CTA
  // per SM; at N = 14, 15 the two-CTA forms spill or lose (profiles/r2/bign/)
  static constexpr int STREAM_T[16] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 2, 2, 0, 0, 0};
  static constexpr int STREAM = STREAM_T[N];
  static constexpr bool GIR = N == 11;
  // Resident CTAs per SM requested from ptxas, from a per-N register target measured on the
  // B200 (0 = no cap, one CTA per SM), capped by shared memory: N = 7 96 registers (10 CTAs per
  // SM; 0.962 vs 0.943 at C3 with 128, profiles/r1b/tune_n7_regs.jsonl); N = 2 80 registers
  // (0.614 vs 0.607, profiles/r1b/last_ab_n2regs_n13pad.jsonl); N = 12 two CTAs per SM with
  // the streamed contractions above; N = 6 96 (aligned rows: 12 CTAs of 56 threads, 80
  // registers; 0.758 vs 0.716 blocked at the same target, 0.695 blocked at 128); N = 13-15 uncapped
  static constexpr int REGS_T[16] = {0, 64, 80, 64, 96, 96, 96, 96, 128, 128, 128, 128, 160, 0, 0, 0};
  static constexpr int REGS = REGS_T[N];
  static constexpr int MINB_REG0 = REGS ? 65536 / (BLOCK * REGS) : 1;
  static constexpr int MINB_REG = MINB_REG0 < 1 ? 1 : (MINB_REG0 > 16 ? 16 : MINB_REG0);
  static constexpr int MINB_SMEM = (int)((227 * 1024) / (SMEM + 1024));
  static constexpr int MINB = MINB_REG < MINB_SMEM ? MINB_REG : (MINB_SMEM < 1 ? 1 : MINB_SMEM);
  // per-element L2 prefetch of G: a gain from N = 6 up, a 1-3% loss below (profiles/r1_tune2.jsonl).
  // 1 = one prefetch.global.L2 per 128-byte line by the element's threads, 2 = one bulk
  // prefetch (cp.async.bulk.prefetch.L2) of the element's whole G range by one thread: fewer
  // LSU instructions, +4..14% at N = 8, 11-15, -5% at N = 7, 10 (profiles/r1b/pf_*.jsonl)
  static constexpr int PFL_T[16] = {0, 0, 0, 0, 0, 0, 1, 1, 2, 1, 1, 2, 2, 2, 2, 2};
  static constexpr int PFL_DEF = PFL_T[N];
  // Folded D from constant memory (uniform-register / constant-bank operands of the DFMAs, no
  // shared-memory broadcast wavefronts) per phase (mask bit 0 P1, 1 P2, 2 P4, 3 P5); 0 = all from
  // shared memory.  Chosen per N from the CG-embedded operator time at the C3 boxes
  // (profiles/r2/dc/insitu_masks.jsonl): all phases +3..9% at N = 2-7, 9, 10, 12 (C2 operator
  // 28.2 -> 27.2 us); N = 14 P2, P4, P5 only (+4%); at N = 8, 11, 15 the constant loads cost
  // registers (spills under the caps) and lose 2-13%; N = 13 P2, P4, P5 only (+5%)
  static constexpr int DC_T[16] = {0, 0, 15, 15, 15, 15, 15, 15, 0, 15, 15, 0, 15, 14, 14, 0};
  static constexpr int DC_DEF = DC_T[N];
};

// Source of the folded matrices: shared memory (warp-uniform broadcast loads, 16-byte pairs) or
// constant memory (DC kernels: the offsets are compile-time after unrolling, so each entry is a
// constant-bank operand of its DFMA -- no load instruction, no L1 data-pipe wavefront).
struct SmemMat {
  const double* __restrict__ p;
  __device__ __forceinline__ double2 pair(int o) const { return *reinterpret_cast<const double2*>(p + o); }
  __device__ __forceinline__ double one(int o) const { return p[o]; }
};
struct ConstMat {
  int base;
  __device__ __forceinline__ double2 pair(int o) const { return make_double2(c_EO[base + o], c_EO[base + o + 1]); }
  __device__ __forceinline__ double one(int o) const { return c_EO[base + o]; }
};

// sum_m C[off + m] v[l][m] for L lines; C is read as 16-byte aligned pairs
template <int CNT, int L, int W, class M>
__device__ __forceinline__ void dot_rows(const M& C, int off, const double (&v)[L][W], double (&acc)[L]) {
#pragma unroll
  for (int m = 0; m + 1 < CNT; m += 2) {
    const double2 c2 = C.pair(off + m);
#pragma unroll
    for (int l = 0; l < L; ++l) {
      acc[l] = fma(c2.x, v[l][m], acc[l]);
      acc[l] = fma(c2.y, v[l][m + 1], acc[l]);
    }
  }
  if constexpr (CNT & 1) {
    const double cl = C.one(off + CNT - 1);
#pragma unroll
    for (int l = 0; l < L; ++l) acc[l] = fma(cl, v[l][CNT - 1], acc[l]);
  }
}

// y[l] = M x[l] for L lines at once (each uniform load of M feeds L multiply-adds).
template <int N, int EPBX, int L, class MS>
__device__ __forceinline__ void eo_apply(const MS& sM, const double (&x)[L][N + 1], double (&y)[L][N + 1]) {
  using S = LinesShape<N, EPBX>;
  constexpr int H = S::H, HE = S::HE, ODD = S::ODD, HE2 = S::HE2, H2 = S::H2;
  constexpr int Me = 0, Mo = H * HE2, Mm = Mo + H * H2;
  double e[L][HE], o[L][H > 0 ? H : 1];
#pragma unroll
  for (int l = 0; l < L; ++l) {
#pragma unroll
    for (int m = 0; m < H; ++m) {
      e[l][m] = x[l][m] + x[l][N - m];
      o[l][m] = x[l][m] - x[l][N - m];
    }
    if constexpr (ODD) e[l][H] = x[l][H];
  }
#pragma unroll
  for (int i = 0; i < H; ++i) {
    double se[L], so[L];
#pragma unroll
    for (int l = 0; l < L; ++l) { se[l] = 0.0; so[l] = 0.0; }
    dot_rows<HE, L, HE>(sM, Me + i * HE2, e, se);
    dot_rows<H, L, (H > 0 ? H : 1)>(sM, Mo + i * H2, o, so);
#pragma unroll
    for (int l = 0; l < L; ++l) {
      y[l][i] = so[l] + se[l];
      y[l][N - i] = so[l] - se[l];
    }
  }
  if constexpr (ODD) {
    double sm[L];
#pragma unroll
    for (int l = 0; l < L; ++l) sm[l] = 0.0;
    dot_rows<H, L, (H > 0 ? H : 1)>(sM, Mm, o, sm);
#pragma unroll
    for (int l = 0; l < L; ++l) y[l][H] = sm[l];
  }
}

// Fused p.Ap (P:217's dot, computed as the element energy): CTA tree sum in shared memory,
// one partial per CTA, the last CTA sums the partials in CTA order (deterministic) and either
// accumulates (more launches of this apply follow) or publishes p.Ap = e + lambda p.p and
// rotates r.r (the bookkeeping a separate p.Ap kernel would do).
__host__ __device__ constexpr int pow2_ceil(int v) { return v <= 1 ? 1 : 2 * pow2_ceil((v + 1) / 2); }

template <int BLOCK>
__device__ __forceinline__ void energy_finish(double en, const AxArgs& a, double* red) {
  __shared__ bool s_last;
  const int t = threadIdx.x;
  red[t] = en;
  __syncthreads();
  constexpr int P2B = pow2_ceil(BLOCK);
#pragma unroll
  for (int h = P2B / 2; h > 0; h >>= 1) {
    if (t < h && t + h < BLOCK) red[t] += red[t + h];
    __syncthreads();
  }
  if (a.e_final == 2) {  // deferred: cg_update_xr_e sums the partials
    if (t == 0) a.e_part[blockIdx.x] = red[0];
    return;
  }
  if (t == 0) {
    a.e_part[blockIdx.x] = red[0];
    __threadfence();
    s_last = (atomicAdd(&a.cg->ticket_e, 1u) == gridDim.x - 1);
  }
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  // last CTA: ordered sum of the partials (fixed strided assignment + fixed tree)
  double v = 0.0;
  const volatile double* pv = a.e_part;
  for (unsigned b = t; b < gridDim.x; b += BLOCK) v += pv[b];
  red[t] = v;
  __syncthreads();
#pragma unroll
  for (int h = P2B / 2; h > 0; h >>= 1) {
    if (t < h && t + h < BLOCK) red[t] += red[t + h];
    __syncthreads();
  }
  if (t == 0) {
    const double tot = red[0];
    CgScalars* s = a.cg;
    s->ticket_e = 0u;
    if (a.e_final) {
      s->pAp = s->e_acc + tot + a.lam_pp * s->pp;
      s->e_acc = 0.0;
      s->rr = s->rr_new;
      if (a.hist) a.hist[s->it] = s->rr_new;
    } else {
      s->e_acc += tot;
    }
  }
}

template <bool CS>
__device__ __forceinline__ double ldG(const double* p) {
  if constexpr (CS) return __ldcs(p);
  else return __ldg(p);
}
template <bool CS>
__device__ __forceinline__ double2 ldG2(const double2* p) {
  if constexpr (CS) return __ldcs(p);
  else return __ldg(p);
}

// ASM: 0 = fused scatter-add into assembled storage (fp64 RED / store); 1 = write y_L per slot
// (deterministic CSR-gather variant); 2 = scattered storage: read u_e from x_L, write y_L.
// Streaming form for L lines at once: the lines are folded in place (x[l][m] <- e_m, x[l][N-m] <- o_m)
// and each output handed to sink(l, i, y) as soon as it is formed -- D is still read once per L
// lines, but no output arrays are kept (large N: 2 lines of 16 in 64 registers instead of 128).
template <int N, int EPBX, int L, class MS, class Sink>
__device__ __forceinline__ void eo_apply_sinkL(const MS& sM, double (&x)[L][N + 1], Sink&& sink) {
  using S = LinesShape<N, EPBX>;
  constexpr int H = S::H, HE = S::HE, ODD = S::ODD, HE2 = S::HE2, H2 = S::H2;
  constexpr int Me = 0, Mo = H * HE2, Mm = Mo + H * H2;
#pragma unroll
  for (int l = 0; l < L; ++l) {
#pragma unroll
    for (int m = 0; m < H; ++m) {
      const double a = x[l][m], b = x[l][N - m];
      x[l][m] = a + b;
      x[l][N - m] = a - b;
    }
  }
#pragma unroll
  for (int i = 0; i < H; ++i) {
    double se[L], so[L];
#pragma unroll
    for (int l = 0; l < L; ++l) { se[l] = 0.0; so[l] = 0.0; }
#pragma unroll
    for (int m = 0; m + 1 < HE; m += 2) {
      const double2 c2 = sM.pair(Me + i * HE2 + m);
#pragma unroll
      for (int l = 0; l < L; ++l) {
        se[l] = fma(c2.x, x[l][m], se[l]);
        se[l] = fma(c2.y, x[l][m + 1], se[l]);
      }
    }
    if constexpr (HE & 1) {
      const double cl = sM.one(Me + i * HE2 + HE - 1);
#pragma unroll
      for (int l = 0; l < L; ++l) se[l] = fma(cl, x[l][HE - 1], se[l]);
    }
#pragma unroll
    for (int m = 0; m + 1 < H; m += 2) {
      const double2 c2 = sM.pair(Mo + i * H2 + m);
#pragma unroll
      for (int l = 0; l < L; ++l) {
        so[l] = fma(c2.x, x[l][N - m], so[l]);
        so[l] = fma(c2.y, x[l][N - m - 1], so[l]);
      }
    }
    if constexpr (H & 1) {
      const double cl = sM.one(Mo + i * H2 + H - 1);
#pragma unroll
      for (int l = 0; l < L; ++l) so[l] = fma(cl, x[l][N - (H - 1)], so[l]);
    }
#pragma unroll
    for (int l = 0; l < L; ++l) {
      sink(l, i, so[l] + se[l]);
      sink(l, N - i, so[l] - se[l]);
    }
  }
  if constexpr (ODD) {
    double sm[L];
#pragma unroll
    for (int l = 0; l < L; ++l) sm[l] = 0.0;
#pragma unroll
    for (int m = 0; m + 1 < H; m += 2) {
      const double2 c2 = sM.pair(Mm + m);
#pragma unroll
      for (int l = 0; l < L; ++l) {
        sm[l] = fma(c2.x, x[l][N - m], sm[l]);
        sm[l] = fma(c2.y, x[l][N - m - 1], sm[l]);
      }
    }
    if constexpr (H & 1) {
      const double cl = sM.one(Mm + H - 1);
#pragma unroll
      for (int l = 0; l < L; ++l) sm[l] = fma(cl, x[l][N - (H - 1)], sm[l]);
    }
#pragma unroll
    for (int l = 0; l < L; ++l) sink(l, H, sm[l]);
  }
}

template <int N, bool HALO, bool MASSB, int PF, int MINB = LinesShape<N>::MINB, int EPBX = 0,
          int PFL = LinesShape<N>::PFL_DEF,
          bool GCS = true, int ASM = 0, bool PFN = false, int DCM = LinesShape<N>::DC_DEF,
          int STREAM = LinesShape<N>::STREAM, bool GIR = LinesShape<N>::GIR>
__global__ void __launch_bounds__(LinesShape<N, EPBX>::BLOCK, MINB)
ax_lines(const AxArgs a) {
  using S = LinesShape<N, EPBX>;
  constexpr int NP = S::NP, NP2 = S::NP2, NP3 = S::NP3, EPB = S::EPB, SLAB = S::SLAB;
  extern __shared__ double smem[];
  const int t = threadIdx.x;
  constexpr bool ALN = S::ALN;
  const int le = ALN ? 0 : t / NP2;
  const int c0 = t - le * NP2;
  // (i,j) for columns, (j,k) for rows, (i,k) for s-lines
  const int ca = ALN ? (t & (S::RW - 1)) : c0 % NP;
  const int cb = ALN ? (t / S::RW) : c0 / NP;
  const int c = ALN ? ca + NP * cb : c0;
  const bool lane_ok = !ALN || ca < NP;  // ALN idle lanes: no shared-memory or global access
  double* s_u = smem + (0 * EPB + le) * SLAB;
  double* s_r = smem + (1 * EPB + le) * SLAB;
  double* s_s = smem + (2 * EPB + le) * SLAB;
  // folded D, D^T: constant memory in the phases of mask DCM (bit 0 P1, 1 P2, 2 P4, 3 P5),
  // a shared-memory copy in the others
  const ConstMat c_D{eo_off(N)}, c_DT{eo_off(N) + S::MAT};
  SmemMat s_D{nullptr}, s_DT{nullptr};
  if constexpr (DCM != 15) {
    double* sd = smem + S::DOFF;
    for (int q = t; q < S::CONST; q += S::BLOCK) sd[q] = __ldg(&g_EO[N][q]);
    s_D = SmemMat{sd};
    s_DT = SmemMat{sd + S::MAT};
  }
  const auto m1 = [&]() { if constexpr (DCM & 1) return c_D; else return s_D; }();
  const auto m2 = [&]() { if constexpr (DCM & 2) return c_D; else return s_D; }();
  const auto m4 = [&]() { if constexpr (DCM & 4) return c_DT; else return s_DT; }();
  const auto m5 = [&]() { if constexpr (DCM & 8) return c_DT; else return s_DT; }();
  const bool interior_ij = (ca > 0 && ca < N && cb > 0 && cb < N);
  double en = 0.0;  // element energy u.(S_e u) (+ lambda u.B u) of this thread's nodes

  if constexpr (PF > 0) {
    if (t == 0)
      for (int w = 0; w < PF; ++w) {
        const int64_t nb = a.e_begin + ((int64_t)blockIdx.x + (int64_t)w * gridDim.x) * EPB;
        if (nb < a.e_end) {
          const int64_t ne = (a.e_end - nb) < EPB ? (a.e_end - nb) : EPB;
          prefetch_l2_bulk(a.G + nb * 6 * NP3, (uint32_t)(ne * 6 * NP3 * sizeof(double)));
          prefetch_l2_bulk(a.idx + nb * NP3, (uint32_t)(ne * NP3 * sizeof(int32_t)));
        }
      }
  }
  __syncthreads();

  // P > 1 tolerance mode: iterations after the device-side stop are no-ops (vec.cuh cg_update_p)
  if (a.cg && a.e_final != 2 && (a.cg->flags & 2)) return;

  for (int64_t base = a.e_begin + (int64_t)blockIdx.x * EPB; base < a.e_end; base += (int64_t)gridDim.x * EPB) {
    if constexpr (PF > 0) {
      if (t == 0) {
        const int64_t nb = base + (int64_t)PF * gridDim.x * EPB;
        if (nb < a.e_end) {
          const int64_t ne = (a.e_end - nb) < EPB ? (a.e_end - nb) : EPB;
          prefetch_l2_bulk(a.G + nb * 6 * NP3, (uint32_t)(ne * 6 * NP3 * sizeof(double)));
          prefetch_l2_bulk(a.idx + nb * NP3, (uint32_t)(ne * NP3 * sizeof(int32_t)));
        }
      }
    }
    const int64_t e = base + le;
    const bool act = (e < a.e_end) && lane_ok;

    // Early L2 prefetch of this element's geometric factors (consumed in P3, after the
    // gather and two barriers) and of the next element's index block (next P1).
    if constexpr (PFL) {
      if (act) {
        // PFN: fetch the NEXT element's G one whole element ahead (the first element at the
        // first iteration); otherwise this element's G at the start of its gather
        const int64_t eg = PFN ? e + (int64_t)gridDim.x * EPB : e;
        auto pf_G = [&](int64_t ee) {
          const char* gb = reinterpret_cast<const char*>(a.G + ee * (6 * NP3));
          if constexpr (PFL == 2) {
            if (c == 0) prefetch_l2_bulk(gb, 48 * NP3);
          } else {
            for (int q = c; q < (6 * NP3 * 8) / 128; q += NP2) prefetch_l2_line(gb + q * 128);
          }
        };
        if (PFN && base == a.e_begin + (int64_t)blockIdx.x * EPB) pf_G(e);
        if (eg < a.e_end) pf_G(eg);
        const int64_t en = e + (int64_t)gridDim.x * EPB;
        if (en < a.e_end) {
          const char* ib = reinterpret_cast<const char*>(a.idx + en * NP3);
          for (int q = c; q < (NP3 * 4 + 127) / 128; q += NP2) prefetch_l2_line(ib + q * 128);
        }
      }
    }

    // ---- P1: gather the (i,j) column (Z x) and the t-derivative in registers
    int32_t gi[NP];
    double gt[1][NP];  // ut, later the G-mixed gt
    {
      double col[1][NP];
#pragma unroll
      for (int k = 0; k < NP; ++k) gi[k] = (act && ASM != 2) ? __ldg(a.idx + e * NP3 + k * NP2 + c) : 0;
#pragma unroll
      for (int k = 0; k < NP; ++k) {
        if constexpr (ASM == 2) col[0][k] = act ? __ldg(a.xh + e * NP3 + k * NP2 + c) : 0.0;  // x_L
        else col[0][k] = act ? load_x<HALO>(a, gi[k]) : 0.0;
        if (lane_ok) s_u[S::at(ca, cb, k)] = col[0][k];
      }
      if constexpr (STREAM >= 1) eo_apply_sinkL<N, EPBX, 1>(m1, col, [&](int, int i, double v) { gt[0][i] = v; });
      else eo_apply<N, EPBX, 1>(m1, col, gt);
    }
    __syncthreads();

    // ---- P2: r-line (row owner (j,k) = (ca,cb)) and s-line ((i,k) = (ca,cb)) gradients
    if (!lane_ok) {
    } else if constexpr (STREAM == 2) {
      double in[2][NP];
#pragma unroll
      for (int m = 0; m < NP; ++m) {
        in[0][m] = s_u[S::at(m, ca, cb)];
        in[1][m] = s_u[S::at(ca, m, cb)];
      }
      eo_apply_sinkL<N, EPBX, 2>(m2, in, [&](int l, int i, double v) {
        if (l == 0) s_r[S::at(i, ca, cb)] = v;
        else s_s[S::at(ca, i, cb)] = v;
      });
    } else if constexpr (STREAM == 1) {
      double in[1][NP];
#pragma unroll
      for (int m = 0; m < NP; ++m) in[0][m] = s_u[S::at(m, ca, cb)];
      eo_apply_sinkL<N, EPBX, 1>(m2, in, [&](int, int i, double v) { s_r[S::at(i, ca, cb)] = v; });
#pragma unroll
      for (int m = 0; m < NP; ++m) in[0][m] = s_u[S::at(ca, m, cb)];
      eo_apply_sinkL<N, EPBX, 1>(m2, in, [&](int, int j, double v) { s_s[S::at(ca, j, cb)] = v; });
    } else {
      double in[2][NP], out[2][NP];
#pragma unroll
      for (int m = 0; m < NP; ++m) {
        in[0][m] = s_u[S::at(m, ca, cb)];
        in[1][m] = s_u[S::at(ca, m, cb)];
      }
      eo_apply<N, EPBX, 2>(m2, in, out);
#pragma unroll
      for (int m = 0; m < NP; ++m) {
        s_r[S::at(m, ca, cb)] = out[0][m];
        s_s[S::at(ca, m, cb)] = out[1][m];
      }
    }
    __syncthreads();

    // ---- P3: metric at the (i,j) column nodes
    if (lane_ok) {
      const double* Ge = a.G + e * (6 * NP3);
#pragma unroll
      for (int k = 0; k < NP; ++k) {
        double grr = 0, grs = 0, grt = 0, gss = 0, gst = 0, gtt = 0;
        if (act) {
          // G is read exactly once per apply: streaming (evict-first) loads keep it from
          // displacing the gathered x / accumulated Ap lines that neighbouring elements reuse
          if constexpr (g_pairs(N)) {
            const double2* g2 = reinterpret_cast<const double2*>(Ge + g_off(true, NP2, k, 0, c));
            const double2 p0 = ldG2<GCS>(g2), p1 = ldG2<GCS>(g2 + NP2), p2 = ldG2<GCS>(g2 + 2 * NP2);
            grr = p0.x; grs = p0.y; grt = p1.x; gss = p1.y; gst = p2.x; gtt = p2.y;
          } else {
            const double* g = Ge + g_off(false, NP2, k, 0, c);
            grr = ldG<GCS>(g); grs = ldG<GCS>(g + NP2); grt = ldG<GCS>(g + 2 * NP2);
            gss = ldG<GCS>(g + 3 * NP2); gst = ldG<GCS>(g + 4 * NP2); gtt = ldG<GCS>(g + 5 * NP2);
          }
        }
        const int o = S::at(ca, cb, k);
        const double ur = s_r[o], us = s_s[o], ut = gt[0][k];
        s_r[o] = grr * ur + grs * us + grt * ut;
        s_s[o] = grs * ur + gss * us + gst * ut;
        gt[0][k] = grt * ur + gst * us + gtt * ut;
      }
    }
    __syncthreads();

    // ---- P4: transposed contractions along r and s lines, in place (each line has one owner)
    if (!lane_ok) {
    } else if constexpr (STREAM == 2) {
      double in[2][NP];
#pragma unroll
      for (int m = 0; m < NP; ++m) {
        in[0][m] = s_r[S::at(m, ca, cb)];
        in[1][m] = s_s[S::at(ca, m, cb)];
      }
      eo_apply_sinkL<N, EPBX, 2>(m4, in, [&](int l, int i, double v) {
        if (l == 0) s_r[S::at(i, ca, cb)] = v;
        else s_s[S::at(ca, i, cb)] = v;
      });
    } else if constexpr (STREAM == 1) {
      double in[1][NP];
#pragma unroll
      for (int m = 0; m < NP; ++m) in[0][m] = s_r[S::at(m, ca, cb)];
      eo_apply_sinkL<N, EPBX, 1>(m4, in, [&](int, int i, double v) { s_r[S::at(i, ca, cb)] = v; });
#pragma unroll
      for (int m = 0; m < NP; ++m) in[0][m] = s_s[S::at(ca, m, cb)];
      eo_apply_sinkL<N, EPBX, 1>(m4, in, [&](int, int j, double v) { s_s[S::at(ca, j, cb)] = v; });
    } else {
      double in[2][NP], out[2][NP];
#pragma unroll
      for (int m = 0; m < NP; ++m) {
        in[0][m] = s_r[S::at(m, ca, cb)];
        in[1][m] = s_s[S::at(ca, m, cb)];
      }
      eo_apply<N, EPBX, 2>(m4, in, out);
#pragma unroll
      for (int m = 0; m < NP; ++m) {
        s_r[S::at(m, ca, cb)] = out[0][m];
        s_s[S::at(ca, m, cb)] = out[1][m];
      }
    }
    __syncthreads();

    // ---- P5: t-direction transposed contraction, sum, assembly Z^T
    if (act) {
      // GIR: the index column is re-read here (L1/L2 hit) instead of held in registers from P1
      int32_t gr[GIR ? NP : 1];
      if constexpr (GIR) {
#pragma unroll
        for (int k = 0; k < NP; ++k) gr[k] = __ldg(a.idx + e * NP3 + k * NP2 + c);
      }
      auto gidx = [&](int k) { if constexpr (GIR) return gr[k]; else return gi[k]; };
      // node k of the (i,j) column: sum the three directions, lambda terms, assembly Z^T
      auto node = [&](int k, double vtk) {
        const int o = S::at(ca, cb, k);
        double out = vtk + s_r[o] + s_s[o];
        const double uk = s_u[o];
        en = fma(uk, out, en);
        if (MASSB) {
          const double lb = a.lam * __ldg(a.B + e * NP3 + k * NP2 + c) * uk;
          out += lb;
          en = fma(uk, lb, en);
        }
        if constexpr (ASM >= 1) {  // y_L per slot, assembled by a CSR (gather-scatter) kernel
          a.yh[e * NP3 + k * NP2 + c] = out;  // y_L
        } else if (interior_ij && k > 0 && k < N) {
          if (!MASSB) out = fma(a.lam, uk, out);  // W = 1 on element-interior nodes
          a.y[gidx(k)] = out;                        // sole contribution: plain store
        } else {
          red_y<HALO>(a, gidx(k), out);
        }
      };
      if constexpr (STREAM >= 1) {
        eo_apply_sinkL<N, EPBX, 1>(m5, gt, [&](int, int k, double v) { node(k, v); });
      } else {
        double vt[1][NP];
        eo_apply<N, EPBX, 1>(m5, gt, vt);
#pragma unroll
        for (int k = 0; k < NP; ++k) node(k, vt[0][k]);
      }
    }
    __syncthreads();
  }
  if (a.cg) energy_finish<S::BLOCK>(en, a, smem);
}

}  // namespace hbk
