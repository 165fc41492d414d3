// Shared definitions of the operator kernels: argument block, the constant-memory D table,
// the halo-aware load/accumulate helpers and the L2 bulk prefetch.
#pragma once
#include <cstdint>

namespace hbk {


__constant__ double c_D[16][256];  // c_D[N][i*(N+1)+j] = D_ij for N = 1..15
// even/odd folded D and D^T per N (layout in ax_lines.cuh LinesShape), written by the host
constexpr int EO_MAX = 272;
__device__ double g_EO[16][EO_MAX];
// Size (doubles) of the folded D | D^T pair of degree N: 2 (H HE2 + H H2 + H2), H = (N+1)/2,
// HE = H + ((N+1) & 1), HE2 / H2 rounded up to even (16-byte row pairs)
__host__ __device__ constexpr int eo_const(int N) {
  return 2 * (((N + 1) / 2) * (((N + 1) / 2 + ((N + 1) & 1)) + ((((N + 1) / 2 + ((N + 1) & 1))) & 1)) +
              ((N + 1) / 2) * ((N + 1) / 2 + (((N + 1) / 2) & 1)) + ((N + 1) / 2 + (((N + 1) / 2) & 1)));
}
__host__ __device__ constexpr int eo_off(int N) { return N <= 1 ? 0 : eo_off(N - 1) + eo_const(N - 1); }
constexpr int EO_TOTAL = eo_off(16);
// the same tables in constant memory, packed per degree: a warp-uniform D entry with a
// compile-time offset becomes a constant-bank operand of the DFMA (no shared-memory wavefront)
__constant__ double c_EO[EO_TOTAL];

// Device-resident CG scalars (alpha, beta are never sent to the host; see vec.cuh)
struct CgScalars {
  double pAp;      // p.Ap (global after allreduce)
  double rr;       // r_j.r_j
  double rr_new;   // r_{j+1}.r_{j+1} (global after allreduce)
  double pp;       // local p.p (for the lambda term of the fused p.Ap)
  double e_acc;    // element-energy accumulator across the operator launches of one apply
  double rz;       // Jacobi PCG: r_j.z_j (z = M^-1 r), the rho of alpha / beta
  double rr_loc;   // r_{j+1}.r_{j+1} from the r update (local; allreduced in place for P > 1),
                   // published as rr_new by the p update
  double pad;
  int32_t it;        // iteration counter j
  uint32_t ticket;   // last-CTA detection, vector kernels
  uint32_t ticket_e; // last-CTA detection, operator energy
  int32_t flags;     // bit 0: CG breakdown detected on the device (tolerance mode);
                     // bit 1: tolerance-mode solve finished (P > 1: later iterations of a chunk are no-ops)
};

struct AxArgs {
  const int32_t* __restrict__ idx;  // [E][NP3] local index into [owned | halo]
  const double* __restrict__ G;     // [E][NP][6 NP2] slab-major, see g_off
  const double* __restrict__ B;     // [E][NP3] (mass mode 1) or null
  const double* __restrict__ x;     // owned values
  const double* __restrict__ xh;    // halo values (HALO); x_L (ASM == 2)
  double* y;                        // owned output (pre-initialised)
  double* yh;                       // halo output accumulator (HALO); y_L per slot (ASM 1, 2)
  // (the struct stays at 128 bytes: a larger kernel parameter block measurably changed the
  //  operator's code generation -- 10% slower at N = 7)
  int64_t e_begin, e_end;           // element range of this launch
  int32_t n_owned;
  int32_t halo_mode;                // HALO kernels: 0 xh / yh arrays; 1 xh / yh hold per-halo-node
                                    // pointers into the owners' p / Ap (IPC direct mode, peer memory)
  double lam;
  // fused p.Ap (CG only; cg == nullptr otherwise): p.Ap = sum_e u_e^T S_e u_e + lambda p.p
  CgScalars* cg;
  double* e_part;   // per-CTA partial energies
  double* hist;     // r.r history (written with the rr rotation by the final launch)
  double lam_pp;    // lambda (mass mode 0) or 0 (mode 1: lambda B is in the element energy)
  int32_t e_final;  // 0: accumulate into e_acc; 1: this launch completes the apply, publish
                    // p.Ap; 2: single-launch apply (P = 1): only write the per-CTA partials,
                    // the x/r update kernel reduces them (no fence/atomic in the operator)
};

// Device layout of the six geometric factors of one element: k-layer slabs, each holding either
// the six factors as separate NP^2 planes, or (g_pairs(N)) three interleaved pairs (rr,rs)
// (rt,ss) (st,tt) per node (i,j): one 16-byte load per pair, a warp's load of a pair is 512
// contiguous bytes.  Pairs measured +2..5% at N = 2, 7, 8 and -2..10% at N = 9, 10, 12, 13
// (profiles/r1b/gp_*.jsonl).  Offset (doubles) of factor f at node (c = i + NP j, k).
__host__ __device__ constexpr bool g_pairs(int N) { return N == 2 || N == 7 || N == 8; }
__host__ __device__ constexpr int g_off(bool pairs, int NP2, int k, int f, int c) {
  return pairs ? ((k * 3 + (f >> 1)) * NP2 + c) * 2 + (f & 1) : (k * 6 + f) * NP2 + c;
}

static_assert(sizeof(AxArgs) == 128, "AxArgs must stay at 128 bytes (see the comment in the struct)");

template <bool HALO>
__device__ __forceinline__ double load_x(const AxArgs& a, int32_t g) {
  if (HALO && g >= a.n_owned) {
    const int32_t h = g - a.n_owned;
    if (a.halo_mode) return *reinterpret_cast<const double* const*>(a.xh)[h];  // owner's p (peer memory)
    return a.xh[h];
  }
  return __ldg(a.x + g);
}

template <bool HALO>
__device__ __forceinline__ void red_y(const AxArgs& a, int32_t g, double v) {
  if (HALO && g >= a.n_owned) {
    const int32_t h = g - a.n_owned;
    if (a.halo_mode) atomicAdd(reinterpret_cast<double* const*>(a.yh)[h], v);  // owner's Ap (peer memory)
    else atomicAdd(a.yh + h, v);
  } else {
    atomicAdd(a.y + g, v);
  }
}

// L2 prefetch of a contiguous byte range by the bulk-copy engine (sm_90+): no registers,
// no shared memory; keeps HBM streaming while the SM works on earlier elements.
// The bulk engine needs a 16-byte aligned start and a multiple-of-16 size: round outwards.
__device__ __forceinline__ void prefetch_l2_bulk(const void* p, uint32_t bytes) {
  const uintptr_t a0 = reinterpret_cast<uintptr_t>(p) & ~uintptr_t(15);
  const uintptr_t a1 = (reinterpret_cast<uintptr_t>(p) + bytes + 15) & ~uintptr_t(15);
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(a0), "r"((uint32_t)(a1 - a0)) : "memory");
}

// Programmatic dependent launch: wait until the preceding kernel of the stream has completed
// and its memory is visible (no-op when the kernel was launched without the PDL attribute).
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

// Per-thread L2 prefetch of one 128-byte line (no registers, no completion tracking).
__device__ __forceinline__ void prefetch_l2_line(const void* p) {
  asm volatile("prefetch.global.L2 [%0];" ::"l"(p));
}

}  // namespace hbk
