// Device side of the C ABI: operator (hb_op_*), CG solve, forcing, dots, NCCL comm,
// loopback groups and the 8:1 streaming calibration.  See include/hipbone_b200.h.
//
// Operator apply schedule (Fig. operator_timeline), P > 1:
//   compute: init y | pack x at shared DOFs            comm: (wait) halo exchange -> xh
//   compute: interior A  (overlaps the halo exchange)
//   compute: (wait halo) halo elements -> y, yh        comm: (wait) assembly exchange yh -> recv
//   compute: interior B  (overlaps the assembly exchange)
//   compute: (wait assembly) y[send_loc] += recv
// P = 1 is one kernel over all elements (plus the lambda-x init, folded into the CG p-update).
// CG: per iteration  op(p) -> dot p.Ap [allreduce] -> x,r update + r.r [allreduce]
// -> p update (writes the next assembly init lambda*p).  No host synchronisation inside the
// loop; fixed-iteration mode is captured once into a CUDA graph and replayed.
#include <cuda.h>  // driver types of the stream memory operations (entry points resolved at run time)
#include <cuda_runtime.h>
#include <nccl.h>

#include <algorithm>
#include <type_traits>
#include <cstdlib>
#include <cmath>
#include <cstring>
#include <map>
#include <memory>
#include <new>
#include <tuple>
#include <vector>

#include "ax_lines.cuh"
#include "ax_vertex.cuh"
#include "internal.h"
#include "vec.cuh"

using hb::set_error;

#define CU_TRY(expr)                                                                      \
  do {                                                                                    \
    cudaError_t _e = (expr);                                                              \
    if (_e != cudaSuccess) {                                                              \
      (void)cudaGetLastError(); /* clear the sticky last-error slot */                    \
      set_error(std::string(__func__) + ": " #expr ": " + cudaGetErrorString(_e));        \
      return (_e == cudaErrorMemoryAllocation) ? HB_ERR_OOM : HB_ERR_CUDA;                \
    }                                                                                     \
  } while (0)

#define NC_TRY(expr)                                                                      \
  do {                                                                                    \
    ncclResult_t _r = (expr);                                                             \
    if (_r != ncclSuccess) {                                                              \
      set_error(std::string(__func__) + ": " #expr ": " + ncclGetErrorString(_r));        \
      return HB_ERR_NCCL;                                                                 \
    }                                                                                     \
  } while (0)

#define HB_TRY(expr)             \
  do {                           \
    int _s = (expr);             \
    if (_s != HB_OK) return _s;  \
  } while (0)

struct hb_comm {
  ncclComm_t nccl = nullptr;
  int P = 1, rank = 0;
  int kind = 0;  // 0: NCCL; 1: IPC peer-memory transport (hb_comm_create_ipc)
};

namespace {

struct DevBuf {
  void* p = nullptr;
  size_t bytes = 0;
  bool own = true;
  ~DevBuf() { if (p && own) cudaFree(p); }
  int alloc(size_t b) {
    if (p && own) cudaFree(p);
    p = nullptr;
    own = true;
    bytes = b;
    if (b == 0) return HB_OK;
    cudaError_t e = cudaMalloc(&p, b);
    if (e != cudaSuccess) { p = nullptr; set_error(std::string("cudaMalloc: ") + cudaGetErrorString(e)); return HB_ERR_OOM; }
    return HB_OK;
  }
  void view(void* ptr, size_t b) {  // non-owning sub-range of an arena
    if (p && own) cudaFree(p);
    p = ptr; bytes = b; own = false;
  }
  template <class T> T* as() const { return reinterpret_cast<T*>(p); }
};

// Launch-shape knobs for A/B measurements exist only in tuning builds (-DHB_TUNE, build.py
// with HB_TUNE=1); the product library ignores the environment.
#ifdef HB_TUNE
const char* tune_env(const char* name) { return getenv(name); }
#else
const char* tune_env(const char*) { return nullptr; }
#endif

struct AxKernel {
  const void* fn = nullptr;
  int block = 0, epb = 0, grid_max = 0;
  size_t smem = 0;
};

template <int N, bool HALO, bool MASSB, int PF, int MINB = hbk::LinesShape<N>::MINB, int EPBX = 0,
          int PFL = hbk::LinesShape<N>::PFL_DEF, bool GCS = true, int ASM = 0, bool PFN = false,
          int DC = hbk::LinesShape<N>::DC_DEF, int STREAM = hbk::LinesShape<N>::STREAM, bool GIR = hbk::LinesShape<N>::GIR>
AxKernel make_lines() {
  AxKernel k;
  k.fn = reinterpret_cast<const void*>(&hbk::ax_lines<N, HALO, MASSB, PF, MINB, EPBX, PFL, GCS, ASM, PFN, DC, STREAM, GIR>);
  k.block = hbk::LinesShape<N, EPBX>::BLOCK;
  k.epb = hbk::LinesShape<N, EPBX>::EPB;
  k.smem = hbk::LinesShape<N, EPBX>::SMEM;
  return k;
}

template <int EPB, bool HALO, bool MASSB, int MINB, int PFB = 1>
AxKernel make_vertex() {
  AxKernel k;
  k.fn = reinterpret_cast<const void*>(&hbk::ax_vertex<EPB, HALO, MASSB, MINB, PFB>);
  k.block = hbk::VertexShape<EPB>::BLOCK;
  k.epb = EPB;
  k.smem = hbk::VertexShape<EPB>::SMEM;
  return k;
}

// N = 1, fused scatter-add: one element per thread (ax_vertex.cuh), 64 elements per CTA
// with an L2 prefetch of G one grid batch ahead (C3: 3.86 ms = 0.86 of peak; no prefetch
// 4.59 ms, line kernel 5.56 ms); tuning builds: HB_N1_LINES=1, HB_N1_EPB=32|64|128, HB_N1_PF=0|1|2
AxKernel pick_vertex(bool halo, bool massb) {
  const char* ev = tune_env("HB_N1_EPB");
  const char* pv = tune_env("HB_N1_PF");
  const int epb = ev ? atoi(ev) : 64, pf = pv ? atoi(pv) : 1;
#define HB_VX(E, M, P) \
  (halo ? (massb ? make_vertex<E, true, true, M, P>() : make_vertex<E, true, false, M, P>()) \
        : (massb ? make_vertex<E, false, true, M, P>() : make_vertex<E, false, false, M, P>()))
  if (epb == 32) return pf == 0 ? HB_VX(32, 16, 0) : pf == 2 ? HB_VX(32, 16, 2) : HB_VX(32, 16, 1);
  if (epb == 128) return pf == 0 ? HB_VX(128, 4, 0) : pf == 2 ? HB_VX(128, 4, 2) : HB_VX(128, 4, 1);
  return pf == 0 ? HB_VX(64, 8, 0) : pf == 2 ? HB_VX(64, 8, 2) : HB_VX(64, 8, 1);
#undef HB_VX
}

constexpr int kLinesPF = 0;  // L2 bulk prefetch distance (grid waves); measured slower on B200

template <int N>
AxKernel pick_ax_n(bool halo, bool massb, int asm_mode) {
  constexpr int M = hbk::LinesShape<N>::MINB;
  if (halo) return massb ? make_lines<N, true, true, kLinesPF>() : make_lines<N, true, false, kLinesPF>();
  constexpr int PL = hbk::LinesShape<N>::PFL_DEF;
  if (asm_mode == 1)
    return massb ? make_lines<N, false, true, kLinesPF, M, 0, PL, true, 1>()
                 : make_lines<N, false, false, kLinesPF, M, 0, PL, true, 1>();
  if (asm_mode == 2) return make_lines<N, false, false, kLinesPF, M, 0, PL, true, 2>();  // mass mode 0 only
  return massb ? make_lines<N, false, true, kLinesPF>() : make_lines<N, false, false, kLinesPF>();
}

#ifdef HB_TUNE
// Tuning build (-DHB_TUNE): per-N launch-shape variants selected with HB_AX_VN / HB_AX_VARIANT.
template <int N, int EPBX, int REGS>
constexpr int tune_minb() {
  using S = hbk::LinesShape<N, EPBX>;
  int r = 65536 / (S::BLOCK * REGS);
  int m = (int)((227 * 1024) / (S::SMEM + 1024));
  r = r < m ? r : m;
  r = r > 16 ? 16 : r;
  return r < 1 ? 1 : r;
}

template <int N>
AxKernel tune_variant(int v) {
  constexpr int NP2 = (N + 1) * (N + 1);
  constexpr int E128 = 128 / NP2 > 0 ? 128 / NP2 : 1;
  constexpr int E256 = 256 / NP2 > 0 ? 256 / NP2 : 1;
  switch (v) {
    case 1: return make_lines<N, false, false, 0, tune_minb<N, E128, 96>(), E128>();
    case 2: return make_lines<N, false, false, 0, tune_minb<N, E256, 96>(), E256>();
    case 3: return make_lines<N, false, false, 0, tune_minb<N, 0, 64>()>();
    case 4: return make_lines<N, false, false, 0, 1>();
    case 5: return make_lines<N, false, false, 0, tune_minb<N, 0, 128>()>();
    case 6: return make_lines<N, false, false, 0, tune_minb<N, E128, 128>(), E128>();
    case 7: return make_lines<N, false, false, 0, hbk::LinesShape<N>::MINB, 0, true, true, 0, true>();  // G one element ahead
    case 8: return make_lines<N, false, false, 0, hbk::LinesShape<N>::MINB, 0, false>();                // no G prefetch
    case 9: return make_lines<N, false, false, 0, tune_minb<N, 0, 112>()>();   // 112 regs
    case 10: return make_lines<N, false, false, 0, tune_minb<N, 0, 96>()>();   // 96 regs
    case 11: return make_lines<N, false, false, 0, tune_minb<N, 0, 80>()>();   // 80 regs
    case 13: return make_lines<N, false, false, 0, hbk::LinesShape<N>::MINB, 0, 2>();  // bulk G of this element
    // folded D from constant memory (DFMA constant-bank operands) per phase mask / from shared memory
#define HB_DCV(MASK) make_lines<N, false, false, 0, hbk::LinesShape<N>::MINB, 0, hbk::LinesShape<N>::PFL_DEF, true, 0, false, MASK>()
    case 30: return HB_DCV(15);
    case 31: return HB_DCV(0);
    case 35: return HB_DCV(9);   // P1 + P5 (single-line phases)
    case 36: return HB_DCV(6);   // P2 + P4 (two-line phases)
    case 37: return HB_DCV(1);
    case 38: return HB_DCV(8);
    case 39: return HB_DCV(14);
#undef HB_DCV
    // large N: two-line streamed contractions (STREAM 2), index re-read in P5 (GIR), register targets
#define HB_SV(ST, GR, REGS) make_lines<N, false, false, 0, tune_minb<N, 0, REGS>(), 0, hbk::LinesShape<N>::PFL_DEF, true, 0, false, hbk::LinesShape<N>::DC_DEF, ST, GR>()
    case 60: return HB_SV(2, false, 255);
    case 61: return HB_SV(2, false, 128);
    case 62: return HB_SV(2, true, 128);
    case 63: return HB_SV(2, true, 168);
    case 64: return HB_SV(2, false, 168);
    case 65: return HB_SV(0, false, 255);
    case 66: return HB_SV(2, true, 96);
    case 67: return HB_SV(2, true, 112);
    case 68: return HB_SV(1, true, 128);
    case 69: return HB_SV(1, false, 128);
    case 70: return HB_SV(1, true, 168);
    case 71: return make_lines<N, false, false, 0, tune_minb<N, 0, 128>(), 0, hbk::LinesShape<N>::PFL_DEF, true, 0, false, 0, 2, true>();
    case 72: return make_lines<N, false, false, 0, tune_minb<N, 0, 128>(), 0, hbk::LinesShape<N>::PFL_DEF, true, 0, false, 0, 1, true>();
    case 73: return make_lines<N, false, false, 0, tune_minb<N, 0, 168>(), 0, hbk::LinesShape<N>::PFL_DEF, true, 0, false, 0, 2, false>();
    // N = 6: the blocked thread mapping (round-1 layout) at the former and the current register target
    case 100: if constexpr (N == 6) return make_lines<N, false, false, 0, tune_minb<N, 1, 128>(), 1>(); else break;
    case 101: if constexpr (N == 6) return make_lines<N, false, false, 0, tune_minb<N, 1, 96>(), 1>(); else break;
    case 74: return HB_SV(0, false, 128);  // round-1 N = 11
    case 75: return HB_SV(1, false, 160);  // round-1 N = 12 (one streamed line)
#undef HB_SV
    case 32: return make_lines<N, false, false, 0, tune_minb<N, 0, 80>(), 0, hbk::LinesShape<N>::PFL_DEF, true, 0, false, 15>();
    case 33: return make_lines<N, false, false, 0, tune_minb<N, 0, 96>(), 0, hbk::LinesShape<N>::PFL_DEF, true, 0, false, 15>();
    case 34: return make_lines<N, false, false, 0, tune_minb<N, 0, 128>(), 0, hbk::LinesShape<N>::PFL_DEF, true, 0, false, 15>();
    default:
      break;
  }
  return make_lines<N, false, false, kLinesPF>();
}

AxKernel pick_ax_variant(int N, int v) {
#ifdef HB_TUNE_N  // one degree only (faster tuning builds)
  if (N == HB_TUNE_N) return tune_variant<HB_TUNE_N>(v);
  return make_lines<7, false, false, 0>();
#endif
  switch (N) {
    case 1: return tune_variant<1>(v);
    case 2: return tune_variant<2>(v);
    case 3: return tune_variant<3>(v);
    case 4: return tune_variant<4>(v);
    case 5: return tune_variant<5>(v);
    case 6: return tune_variant<6>(v);
    case 7: return tune_variant<7>(v);
    case 8: return tune_variant<8>(v);
    case 9: return tune_variant<9>(v);
    case 10: return tune_variant<10>(v);
    case 11: return tune_variant<11>(v);
    case 12: return tune_variant<12>(v);
    case 13: return tune_variant<13>(v);
    case 14: return tune_variant<14>(v);
    default: return tune_variant<15>(v);
  }
}
#endif

AxKernel pick_ax(int N, bool halo, bool massb, int asm_mode = 0) {
#ifdef HB_TUNE
  if (!halo && !massb && asm_mode == 0) {
    const char* v = getenv("HB_AX_VARIANT");
    const char* vn = getenv("HB_AX_VN");
    if (v && atoi(v) > 0 && vn && atoi(vn) == N) return pick_ax_variant(N, atoi(v));
  }
#endif
  if (N == 1 && asm_mode == 0) {
    const char* l = tune_env("HB_N1_LINES");
    if (!(l && l[0] == '1')) return pick_vertex(halo, massb);
  }
  switch (N) {
    case 1: return pick_ax_n<1>(halo, massb, asm_mode);
    case 2: return pick_ax_n<2>(halo, massb, asm_mode);
    case 3: return pick_ax_n<3>(halo, massb, asm_mode);
    case 4: return pick_ax_n<4>(halo, massb, asm_mode);
    case 5: return pick_ax_n<5>(halo, massb, asm_mode);
    case 6: return pick_ax_n<6>(halo, massb, asm_mode);
    case 7: return pick_ax_n<7>(halo, massb, asm_mode);
    case 8: return pick_ax_n<8>(halo, massb, asm_mode);
    case 9: return pick_ax_n<9>(halo, massb, asm_mode);
    case 10: return pick_ax_n<10>(halo, massb, asm_mode);
    case 11: return pick_ax_n<11>(halo, massb, asm_mode);
    case 12: return pick_ax_n<12>(halo, massb, asm_mode);
    case 13: return pick_ax_n<13>(halo, massb, asm_mode);
    case 14: return pick_ax_n<14>(halo, massb, asm_mode);
    default: return pick_ax_n<15>(halo, massb, asm_mode);
  }
}

// packed host G [E][NP3][6] -> device layout [E][NP][6 NP2] (hbk::g_off)
__global__ void relayout_G(const double* __restrict__ src, double* __restrict__ dst, int64_t E, int NP) {
  const int NP2 = NP * NP, NP3 = NP2 * NP;
  const int64_t total = E * NP3;
  for (int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; s < total; s += (int64_t)gridDim.x * blockDim.x) {
    int64_t e = s / NP3;
    int n = (int)(s - e * NP3);
    int k = n / NP2, c = n - k * NP2;
    for (int f = 0; f < 6; ++f) dst[e * 6 * NP3 + hbk::g_off(hbk::g_pairs(NP - 1), NP2, k, f, c)] = src[s * 6 + f];
  }
}

// default box geometry written directly in device layout
__global__ void box_G(double* __restrict__ dst, int64_t E, int N, double grr, double gss, double gtt) {
  const int NP = N + 1, NP2 = NP * NP, NP3 = NP2 * NP;
  const int64_t total = E * NP3;
  for (int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; s < total; s += (int64_t)gridDim.x * blockDim.x) {
    int64_t e = s / NP3;
    int n = (int)(s - e * NP3);
    int k = n / NP2, c = n - k * NP2;
    int i = c % NP, j = c / NP;
    double wq = hbk::c_D[0][i] * hbk::c_D[0][j] * hbk::c_D[0][k];  // weights staged in c_D[0]
    double* d = dst + e * 6 * NP3;
    const bool gp = hbk::g_pairs(N);
    d[hbk::g_off(gp, NP2, k, 0, c)] = wq * grr; d[hbk::g_off(gp, NP2, k, 1, c)] = 0.0; d[hbk::g_off(gp, NP2, k, 2, c)] = 0.0;
    d[hbk::g_off(gp, NP2, k, 3, c)] = wq * gss; d[hbk::g_off(gp, NP2, k, 4, c)] = 0.0; d[hbk::g_off(gp, NP2, k, 5, c)] = wq * gtt;
  }
}

int g_num_sms = 0;
int num_sms() {
  if (g_num_sms == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&g_num_sms, cudaDevAttrMultiProcessorCount, dev);
    if (g_num_sms <= 0) g_num_sms = 148;
  }
  return g_num_sms;
}

int vec_grid(int64_t n) {
  int64_t need = (n / 2 + hbk::VEC_BLOCK - 1) / hbk::VEC_BLOCK;
  int64_t cap = (int64_t)num_sms() * 2;  // 2 x 512-thread CTAs per SM: few partials, cheap last-CTA tickets
  return (int)std::max<int64_t>(1, std::min<int64_t>(need, cap));
}

}  // namespace

struct hb_op {
  hb_sizes sz{};
  int N = 0, NP3 = 0;
  int mass_mode = 0;
  double lam = 1.0;
  hb_comm* comm = nullptr;
  bool grouped = false;
  int64_t nA = 0, nH = 0, nB = 0;
  // device data
  DevBuf arena;  // [idx | r | p | Ap | xs]: the data every CG iteration re-reads besides G
  DevBuf idx, G, B, owned_gid;
  DevBuf r, p, Ap, xs, partials, e_part, pp_part, rz_part, invd, scal, hist, dot_out, dot_ticket;
  bool jacobi = false;  // Jacobi-preconditioned CG (P = 1, fused path)
  bool tol_device_loop = true;  // tolerance mode as one graph with a WHILE node (P = 1)
  bool graph_ok = true;         // P > 1 NCCL: false once capturing the communicator's calls failed
  // P > 1 tolerance mode: the stop test taken on the device by cg_update_p (eps < 0: none)
  double tol_eps = -1.0;
  int32_t tol_max = INT32_MAX;
  bool timing_vec_only = false; // measurement hook: fixed-mode CG without the operator launches
  int variant = 0;      // 0: fused scatter-add (fp64 RED); 1: y_L + CSR gather (deterministic), P = 1
  DevBuf yL, csr_ptr, csr_slots;
  // NekBone scattered storage (NEXT #4): local vectors of length N_L and the weights W
  bool scat_mode = false;  // operator launches read x_L (sL_p) and write y_L
  DevBuf sL_x, sL_r, sL_p, sL_w, sW;
  int fused_grid = 0;  // > 0: P = 1 vector updates in one cooperative kernel of this grid
  hbk::CondTest cond_test = {0, 0.0, 0, 0};  // set while the tolerance graph's WHILE body is captured
  const void* fused_fn = nullptr;  // cg_update_fused<U> instance (U double2 per thread per batch)
  const void* fused_fn_cond = nullptr;  // the same with the tolerance-mode loop test (WHILE condition)
  bool pdl = false;    // P = 1 CG kernels use programmatic dependent launch (env HB_PDL=0 disables)
  DevBuf xh, yh, send_loc, send_buf, recv_buf;
  std::vector<int32_t> nbr;
  std::vector<int64_t> soff, scnt, roff, rcnt;
  int64_t n_send = 0;
  int last_grid = 0;  // grid of the last operator launch (number of energy partials, P = 1)
  AxKernel ax_plain, ax_halo, ax_yl, ax_scat;  // ax_yl / ax_scat picked on first use
  cudaStream_t comm_stream = nullptr;
  cudaStream_t cap_stream = nullptr;  // private stream for graph capture (the legacy stream cannot be captured)
  cudaStream_t cap_stream2 = nullptr; // captures the body of the tolerance-mode WHILE node
  cudaEvent_t ev_cap = nullptr;
  cudaEvent_t ev_pack = nullptr, ev_halo = nullptr, ev_haloel = nullptr, ev_gather = nullptr;
  cudaEvent_t ev_red = nullptr, ev_red_done = nullptr;
  // profiling
  bool profiling = false;
  int prof_stride = 1;      // time every prof_stride-th operator launch
  int64_t prof_seq = 0;     // operator launches seen since profiling was (re)enabled
  std::vector<std::pair<cudaEvent_t, cudaEvent_t>> prof_events;
  size_t prof_used = 0;
  bool last_timed = false;  // the last operator launch was timed: time this iteration's vector kernels too
  struct Timer {
    std::vector<std::pair<cudaEvent_t, cudaEvent_t>> ev;
    size_t used = 0;
  } t_xr, t_p;  // CG vector phases (x/r update, p update)
  int64_t launches = 0;
  // fixed-mode graph cache
  struct GraphKey {
    int32_t K; const double* b; double* x; bool prof; bool vec_only; cudaStream_t st;
    bool operator<(const GraphKey& o) const {
      return std::tie(K, b, x, prof, vec_only, st) < std::tie(o.K, o.b, o.x, o.prof, o.vec_only, o.st);
    }
  };
  struct GraphVal { cudaGraphExec_t exec; int64_t launches; size_t prof_events, prof_xr, prof_p; };
  std::map<GraphKey, GraphVal> graphs;
  struct TolKey {
    int32_t K; const double* b; double* x; double eps; cudaStream_t st;
    bool operator<(const TolKey& o) const { return std::tie(K, b, x, eps, st) < std::tie(o.K, o.b, o.x, o.eps, o.st); }
  };
  std::map<TolKey, GraphVal> tol_graphs;  // tolerance mode, one CUDA graph with a WHILE node
  std::map<TolKey, GraphVal> chunk_graphs;  // P > 1 tolerance mode: a chunk of predicated iterations
  std::map<std::tuple<int32_t, const double*, double*>, GraphVal> scat_graphs;  // scattered-storage CG
  double* host_scal = nullptr;  // pinned CgScalars mirror
  // IPC transport (comm kind 1): peer mappings of the buffers this rank writes into
  struct IpcPeer {
    double* xh = nullptr;      // peer's halo receive buffer (+ xh_off: the segment from this rank)
    double* recv = nullptr;    // peer's assembly receive buffer (+ recv_off)
    uint32_t* flags = nullptr; // peer's mailbox flags [5][P]
    double* vals = nullptr;    // peer's mailbox allreduce slots [2][P]
    int64_t xh_off = 0, recv_off = 0;
  };
  bool ipc_ready = false;
  DevBuf mbox, ipc_tab;  // mailbox; device tables of the P vals / AR-flag pointers
  std::vector<IpcPeer> peers;
  std::vector<void*> ipc_opened;
  uint32_t apply_seq = 0, ar_seq = 0;
  // IPC direct mode (CG): the halo-element kernel reads the owners' p and scatter-adds into
  // the owners' Ap through per-halo-node peer pointers -- no exchange, no pack / unpack
  bool ipc_direct = true;
  DevBuf hx_tab, hy_tab;   // [n_halo] pointers into the owners' p / Ap
  uint32_t iter_seq = 0;   // direct-mode CG iterations so far (RDY / DONE flag values)
  int halo_mode_now = 0;   // launch_ax: pass the pointer tables to the HALO kernel
  ~hb_op() {
    for (void* p : ipc_opened) cudaIpcCloseMemHandle(p);
    for (auto& kv : graphs) cudaGraphExecDestroy(kv.second.exec);
    for (auto& pr : prof_events) { cudaEventDestroy(pr.first); cudaEventDestroy(pr.second); }
    for (Timer* tm : {&t_xr, &t_p})
      for (auto& pr : tm->ev) { cudaEventDestroy(pr.first); cudaEventDestroy(pr.second); }
    if (comm_stream) cudaStreamDestroy(comm_stream);
    if (cap_stream) cudaStreamDestroy(cap_stream);
    if (cap_stream2) cudaStreamDestroy(cap_stream2);
    for (auto& kv : tol_graphs) cudaGraphExecDestroy(kv.second.exec);
    for (auto& kv : chunk_graphs) cudaGraphExecDestroy(kv.second.exec);
    for (auto& kv : scat_graphs) cudaGraphExecDestroy(kv.second.exec);
    if (ev_cap) cudaEventDestroy(ev_cap);
    for (cudaEvent_t e : {ev_pack, ev_halo, ev_haloel, ev_gather, ev_red, ev_red_done}) if (e) cudaEventDestroy(e);
    if (host_scal) cudaFreeHost(host_scal);
  }
};

namespace {

// timing event: an external event node while the stream is being captured, else a plain record
cudaError_t record_event(cudaEvent_t ev, cudaStream_t st) {
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  cudaError_t e = cudaStreamIsCapturing(st, &cs);
  if (e != cudaSuccess) return e;
  return cs == cudaStreamCaptureStatusActive ? cudaEventRecordWithFlags(ev, st, cudaEventRecordExternal)
                                             : cudaEventRecord(ev, st);
}

// dynamic shared memory opt-in and the persistent grid size (resident CTAs x SMs)
int prepare_kernel(AxKernel& k) {
  int nb = 0;
  CU_TRY(cudaFuncSetAttribute(k.fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)k.smem));
  CU_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, k.fn, k.block, k.smem));
  k.grid_max = std::max(1, nb) * num_sms();
  return HB_OK;
}

int launch_ax(hb_op* op, const AxKernel& k, int64_t e0, int64_t e1, const double* x, double* y, cudaStream_t st,
              bool energy = false, bool final_launch = false) {
  if (e1 <= e0) return HB_OK;
  hbk::AxArgs a;
  a.idx = op->idx.as<int32_t>();
  a.G = op->G.as<double>();
  a.B = op->B.as<double>();
  a.x = x;
  a.xh = op->xh.as<double>();
  a.y = y;
  a.yh = op->yh.as<double>();
  if (op->variant == 1 || op->scat_mode) a.yh = op->yL.as<double>();  // ASM >= 1 kernels write y_L there
  if (op->scat_mode) a.xh = op->sL_p.as<double>();                     // ASM == 2 reads x_L there
  a.e_begin = e0; a.e_end = e1;
  a.n_owned = (int32_t)op->sz.n_owned;
  a.halo_mode = 0;
  if (op->halo_mode_now) {
    a.halo_mode = 1;
    a.xh = op->hx_tab.as<double>();
    a.yh = op->hy_tab.as<double>();
  }
  a.lam = op->lam;
  a.cg = energy ? op->scal.as<hbk::CgScalars>() : nullptr;
  a.e_part = op->e_part.as<double>();
  a.hist = op->hist.as<double>();
  a.lam_pp = op->mass_mode == 0 ? op->lam : 0.0;
  a.e_final = final_launch ? ((op->comm && op->comm->P > 1) || op->grouped ? 1 : 2) : 0;
  int64_t groups = (e1 - e0 + k.epb - 1) / k.epb;
  int grid = (int)std::min<int64_t>(groups, (int64_t)k.grid_max);

  if (energy && final_launch) op->last_grid = grid;
  void* args[] = {&a};
  cudaEvent_t e_start = nullptr, e_stop = nullptr;
  const bool timed = op->profiling && (op->prof_seq++ % op->prof_stride == 0);
  op->last_timed = timed;
  if (timed) {
    if (op->prof_used >= op->prof_events.size()) {
      cudaEvent_t s0, s1;
      CU_TRY(cudaEventCreate(&s0));
      CU_TRY(cudaEventCreate(&s1));
      op->prof_events.push_back({s0, s1});
    }
    e_start = op->prof_events[op->prof_used].first;
    e_stop = op->prof_events[op->prof_used].second;
    op->prof_used++;
    CU_TRY(record_event(e_start, st));
  }
  CU_TRY(cudaLaunchKernel(k.fn, dim3(grid), dim3(k.block), args, k.smem, st));
  op->launches++;
  if (timed) CU_TRY(record_event(e_stop, st));
  return HB_OK;
}

// bracket a vector phase with events when the iteration's operator launch was timed
int phase_event(hb_op* op, hb_op::Timer& tm, bool start, cudaStream_t st) {
  if (!op->last_timed) return HB_OK;
  if (start) {
    if (tm.used >= tm.ev.size()) {
      cudaEvent_t s0, s1;
      CU_TRY(cudaEventCreate(&s0));
      CU_TRY(cudaEventCreate(&s1));
      tm.ev.push_back({s0, s1});
    }
    CU_TRY(record_event(tm.ev[tm.used].first, st));
  } else {
    CU_TRY(record_event(tm.ev[tm.used].second, st));
    tm.used++;
  }
  return HB_OK;
}

// --- IPC transport (comm kind 1).  Every rank maps, through CUDA IPC,
// the mailbox of every peer and the halo / assembly receive buffers of its neighbours.  The
// sender copies straight into the receiver's buffer (NVLink copy engine across GPUs) and then
// raises a 32-bit sequence flag in the receiver's mailbox (cuStreamWriteValue32, fenced); the
// receiver's stream waits on it (cuStreamWaitValue32 GEQ).  Per directed neighbour pair four
// flags order one apply s:  HD (halo data in your xh, = s), HF (my xh is consumed, = s),
// AD (assembly data in your recv, = s), AF (my recv is consumed, = s - 1, raised at the start
// of the next apply).  Allreduce: every rank stores its value into slot [s & 1][me] of every
// mailbox and raises AR = s; two slots suffice because no rank can start allreduce s + 2
// before every rank has finished s (it needs their s + 1 values, pushed after their sum of s).
// Direct mode (CG, hb_op_set_ipc_direct): RDY (owner's p and Ap = lambda p of iteration it are
// written, = it) and DONE (sharer's halo elements of iteration it have read p and added into
// Ap, = it) replace both exchanges.
// Mailbox layout: uint32 flags[7][P] (indexed by source rank), then double vals[2][P].
enum { F_HD = 0, F_HF = 1, F_AD = 2, F_AF = 3, F_AR = 4, F_RDY = 5, F_DONE = 6, F_KINDS = 7 };
size_t mbox_vals_off(int P) { return ((size_t)F_KINDS * P * 4 + 255) & ~size_t(255); }
size_t mbox_bytes(int P) { return mbox_vals_off(P) + (size_t)2 * P * 8; }

typedef CUresult (*PfnValue32)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);
PfnValue32 g_wait32 = nullptr, g_write32 = nullptr;

int load_memops() {
  if (g_wait32 && g_write32) return HB_OK;
  cudaDriverEntryPointQueryResult q1 = cudaDriverEntryPointSymbolNotFound, q2 = cudaDriverEntryPointSymbolNotFound;
  CU_TRY(cudaGetDriverEntryPointByVersion("cuStreamWaitValue32", (void**)&g_wait32, 12000, cudaEnableDefault, &q1));
  CU_TRY(cudaGetDriverEntryPointByVersion("cuStreamWriteValue32", (void**)&g_write32, 12000, cudaEnableDefault, &q2));
  if (q1 != cudaDriverEntryPointSuccess || q2 != cudaDriverEntryPointSuccess || !g_wait32 || !g_write32) {
    g_wait32 = g_write32 = nullptr;
    set_error("IPC transport: stream memory operations unavailable in this driver");
    return HB_ERR_CUDA;
  }
  return HB_OK;
}

int mem_wait(cudaStream_t st, const uint32_t* addr, uint32_t v) {
  CUresult r = g_wait32((CUstream)st, (CUdeviceptr)addr, v, CU_STREAM_WAIT_VALUE_GEQ);
  if (r != CUDA_SUCCESS) { set_error("cuStreamWaitValue32 failed (CUresult " + std::to_string((int)r) + ")"); return HB_ERR_CUDA; }
  return HB_OK;
}

int mem_signal(cudaStream_t st, uint32_t* addr, uint32_t v) {
  CUresult r = g_write32((CUstream)st, (CUdeviceptr)addr, v, CU_STREAM_WRITE_VALUE_DEFAULT);  // fenced
  if (r != CUDA_SUCCESS) { set_error("cuStreamWriteValue32 failed (CUresult " + std::to_string((int)r) + ")"); return HB_ERR_CUDA; }
  return HB_OK;
}

bool is_ipc(const hb_op* op) { return op->comm && op->comm->kind == 1; }

// kind 0: halo exchange (owners push x at shared DOFs into the sharers' xh);
// kind 1: assembly exchange (sharers push their halo partial sums yh into the owners' recv).
int ipc_exchange(hb_op* op, int kind, cudaStream_t cs) {
  const int P = op->comm->P, me = op->comm->rank;
  uint32_t* own = op->mbox.as<uint32_t>();
  auto own_flag = [&](int q, int k) { return own + k * P + q; };
  auto peer_flag = [&](int q, int k) { return op->peers[q].flags + k * P + me; };
  if (kind == 0) {
    const uint32_t s = ++op->apply_seq;
    for (size_t i = 0; i < op->nbr.size(); ++i) {
      if (!op->scnt[i]) continue;
      const int q = op->nbr[i];
      HB_TRY(mem_signal(cs, peer_flag(q, F_AF), s - 1));  // the previous apply's recv from q is unpacked
      HB_TRY(mem_wait(cs, own_flag(q, F_HF), s - 1));     // q has consumed the previous halo data
      CU_TRY(cudaMemcpyAsync(op->peers[q].xh + op->peers[q].xh_off, op->send_buf.as<double>() + op->soff[i],
                             op->scnt[i] * 8, cudaMemcpyDeviceToDevice, cs));
      HB_TRY(mem_signal(cs, peer_flag(q, F_HD), s));
    }
    for (size_t i = 0; i < op->nbr.size(); ++i)
      if (op->rcnt[i]) HB_TRY(mem_wait(cs, own_flag(op->nbr[i], F_HD), s));
    return HB_OK;
  }
  const uint32_t s = op->apply_seq;
  for (size_t i = 0; i < op->nbr.size(); ++i) {
    if (!op->rcnt[i]) continue;
    const int q = op->nbr[i];
    HB_TRY(mem_signal(cs, peer_flag(q, F_HF), s));      // halo elements done: xh from q consumed
    HB_TRY(mem_wait(cs, own_flag(q, F_AF), s - 1));     // q has unpacked the previous contribution
    CU_TRY(cudaMemcpyAsync(op->peers[q].recv + op->peers[q].recv_off, op->yh.as<double>() + op->roff[i],
                           op->rcnt[i] * 8, cudaMemcpyDeviceToDevice, cs));
    HB_TRY(mem_signal(cs, peer_flag(q, F_AD), s));
  }
  for (size_t i = 0; i < op->nbr.size(); ++i)
    if (op->scnt[i]) HB_TRY(mem_wait(cs, own_flag(op->nbr[i], F_AD), s));
  return HB_OK;
}

int ipc_allreduce(hb_op* op, double* v, cudaStream_t st) {
  const int P = op->comm->P, me = op->comm->rank;
  const uint32_t s = ++op->ar_seq;
  const int slot = (int)(s & 1);
  double* const* vt = op->ipc_tab.as<double*>();
  uint32_t* const* ft = reinterpret_cast<uint32_t* const*>(vt + P);
  hbk::ipc_push_kernel<<<1, 32, 0, st>>>(v, vt, ft, P, me, slot, s);
  op->launches++;
  CU_TRY(cudaGetLastError());
  uint32_t* own = op->mbox.as<uint32_t>();
  for (int q = 0; q < P; ++q)
    if (q != me) HB_TRY(mem_wait(st, own + F_AR * P + q, s));
  double* vals = reinterpret_cast<double*>(op->mbox.as<char>() + mbox_vals_off(P));
  hbk::ipc_sum_kernel<<<1, 1, 0, st>>>(vals + slot * P, P, v);
  op->launches++;
  CU_TRY(cudaGetLastError());
  return HB_OK;
}

bool direct_mode(const hb_op* op) { return is_ipc(op) && op->comm->P > 1 && op->ipc_direct; }

// owners of this rank's halo nodes (rcnt > 0) / sharers of its owned nodes (scnt > 0)
int ipc_signal_ready(hb_op* op, cudaStream_t st) {  // p and Ap init of the next iteration written
  const int P = op->comm->P, me = op->comm->rank;
  for (size_t i = 0; i < op->nbr.size(); ++i)
    if (op->scnt[i]) HB_TRY(mem_signal(st, op->peers[op->nbr[i]].flags + F_RDY * P + me, op->iter_seq + 1));
  return HB_OK;
}

int allreduce_sum(hb_op* op, double* v, cudaStream_t st) {
  if (!op->comm || op->comm->P == 1) return HB_OK;
  if (is_ipc(op)) return ipc_allreduce(op, v, st);
  NC_TRY(ncclAllReduce(v, v, 1, ncclFloat64, ncclSum, op->comm->nccl, st));
  return HB_OK;
}

// --- staged apply (shared by the single-op path and loopback groups)
int stage_init(hb_op* op, const double* x, double* y, bool init_y, cudaStream_t st) {
  const int64_t n = op->sz.n_owned;
  if (init_y) {
    hbk::vec_scale<<<vec_grid(2 * n), hbk::VEC_BLOCK, 0, st>>>(x, y, n, op->mass_mode == 0 ? op->lam : 0.0);
    op->launches++;
  }
  if (op->sz.n_halo > 0) CU_TRY(cudaMemsetAsync(op->yh.p, 0, op->sz.n_halo * 8, st));
  if (op->n_send > 0) {
    hbk::pack_kernel<<<vec_grid(2 * op->n_send), hbk::VEC_BLOCK, 0, st>>>(x, op->send_loc.as<int32_t>(),
                                                                       op->send_buf.as<double>(), op->n_send);
    op->launches++;
  }
  CU_TRY(cudaGetLastError());
  return HB_OK;
}

int stage_unpack(hb_op* op, double* y, cudaStream_t st) {
  if (op->n_send > 0) {
    hbk::unpack_add_kernel<<<vec_grid(2 * op->n_send), hbk::VEC_BLOCK, 0, st>>>(y, op->send_loc.as<int32_t>(),
                                                                             op->recv_buf.as<double>(), op->n_send);
    op->launches++;
  }
  CU_TRY(cudaGetLastError());
  return HB_OK;
}

// Point-to-point messages of the two exchanges of one apply.  The halo segment of
// the extended vector is the receive buffer of the halo exchange and the send buffer of the
// assembly exchange (zero copy).  Both transports (NCCL, loopback) consume these lists.
struct Msg {
  double* buf;
  int64_t count;
  int peer;
};
void halo_msgs(hb_op* op, std::vector<Msg>& sends, std::vector<Msg>& recvs) {
  sends.clear(); recvs.clear();
  for (size_t q = 0; q < op->nbr.size(); ++q) {
    if (op->scnt[q]) sends.push_back({op->send_buf.as<double>() + op->soff[q], op->scnt[q], op->nbr[q]});
    if (op->rcnt[q]) recvs.push_back({op->xh.as<double>() + op->roff[q], op->rcnt[q], op->nbr[q]});
  }
}
void assembly_msgs(hb_op* op, std::vector<Msg>& sends, std::vector<Msg>& recvs) {
  sends.clear(); recvs.clear();
  for (size_t q = 0; q < op->nbr.size(); ++q) {
    if (op->rcnt[q]) sends.push_back({op->yh.as<double>() + op->roff[q], op->rcnt[q], op->nbr[q]});
    if (op->scnt[q]) recvs.push_back({op->recv_buf.as<double>() + op->soff[q], op->scnt[q], op->nbr[q]});
  }
}

int nccl_exchange(hb_op* op, const std::vector<Msg>& sends, const std::vector<Msg>& recvs, cudaStream_t cs) {
  NC_TRY(ncclGroupStart());
  for (const Msg& m : sends) NC_TRY(ncclSend(m.buf, m.count, ncclFloat64, m.peer, op->comm->nccl, cs));
  for (const Msg& m : recvs) NC_TRY(ncclRecv(m.buf, m.count, ncclFloat64, m.peer, op->comm->nccl, cs));
  NC_TRY(ncclGroupEnd());
  return HB_OK;
}

// Per-rank phases of the split apply, shared by the NCCL path and loopback groups.
// `exchange(kind, cs)` moves the messages of the halo (kind 0) or assembly (kind 1) exchange
// on the communication stream cs; ev_pack / ev_haloel mark when this rank's send data is ready.
template <class Exchange>
int rank_phase_halo(hb_op* op, const double* x, double* y, cudaStream_t st, cudaStream_t cs, bool energy, int last,
                    Exchange&& exchange) {
  HB_TRY(exchange(0, cs));
  CU_TRY(cudaEventRecord(op->ev_halo, cs));
  HB_TRY(launch_ax(op, op->ax_plain, 0, op->nA, x, y, st, energy, last == 0));                  // interior A
  CU_TRY(cudaStreamWaitEvent(st, op->ev_halo, 0));
  HB_TRY(launch_ax(op, op->ax_halo, op->nA, op->nA + op->nH, x, y, st, energy, last == 1));     // halo elements
  CU_TRY(cudaEventRecord(op->ev_haloel, st));
  return HB_OK;
}

template <class Exchange>
int rank_phase_assembly(hb_op* op, const double* x, double* y, cudaStream_t st, cudaStream_t cs, bool energy,
                        int last, Exchange&& exchange) {
  CU_TRY(cudaStreamWaitEvent(cs, op->ev_haloel, 0));
  HB_TRY(exchange(1, cs));
  CU_TRY(cudaEventRecord(op->ev_gather, cs));
  HB_TRY(launch_ax(op, op->ax_plain, op->nA + op->nH, op->sz.E_local, x, y, st, energy, last == 2));  // interior B
  CU_TRY(cudaStreamWaitEvent(st, op->ev_gather, 0));
  return stage_unpack(op, y, st);
}

int last_launch(const hb_op* op) {  // the last non-empty launch publishes p.Ap
  const int64_t nB = op->sz.E_local - op->nA - op->nH;
  return nB > 0 ? 2 : (op->nH > 0 ? 1 : 0);
}

// Direct-mode operator of a CG iteration (IPC, P > 1): Ap += A p with Ap = lambda p already
// written by the p update.  Interior elements first (they overlap the neighbours' progress),
// then -- once every owner of a halo node has published p (RDY) -- the halo elements, which
// read the owners' p and RED into the owners' Ap over peer memory; finally wait until every
// sharer of an owned node has done the same (DONE) before the vector update reads Ap.
int direct_apply(hb_op* op, cudaStream_t st) {
  const int P = op->comm->P, me = op->comm->rank;
  const uint32_t it = ++op->iter_seq;
  const int64_t E = op->sz.E_local, a0 = op->nA, h0 = op->nA, h1 = op->nA + op->nH;
  const int last = op->nH > 0 ? 1 : (E - h1 > 0 ? 2 : 0);
  const double* p = op->p.as<double>();
  double* Ap = op->Ap.as<double>();
  uint32_t* own = op->mbox.as<uint32_t>();
  HB_TRY(launch_ax(op, op->ax_plain, 0, a0, p, Ap, st, true, last == 0));
  HB_TRY(launch_ax(op, op->ax_plain, h1, E, p, Ap, st, true, last == 2));
  for (size_t i = 0; i < op->nbr.size(); ++i)
    if (op->rcnt[i]) HB_TRY(mem_wait(st, own + F_RDY * P + op->nbr[i], it));
  op->halo_mode_now = 1;
  const int hs = launch_ax(op, op->ax_halo, h0, h1, p, Ap, st, true, last == 1);
  op->halo_mode_now = 0;
  HB_TRY(hs);
  for (size_t i = 0; i < op->nbr.size(); ++i)
    if (op->rcnt[i]) HB_TRY(mem_signal(st, op->peers[op->nbr[i]].flags + F_DONE * P + me, it));
  for (size_t i = 0; i < op->nbr.size(); ++i)
    if (op->scnt[i]) HB_TRY(mem_wait(st, own + F_DONE * P + op->nbr[i], it));
  return HB_OK;
}

// y = A x for one op (P = 1, or P > 1 with NCCL).  init_y=false: y already holds the
// assembly initialisation (lambda x or 0), as written by the CG p-update.  energy=true (CG):
// the operator launches also reduce p.Ap (element energy) into the CG scalars.
int apply_internal(hb_op* op, const double* x, double* y, bool init_y, cudaStream_t st, bool energy = false) {
  const int64_t E = op->sz.E_local;
  const bool multi = op->comm && op->comm->P > 1;
  if (!multi) {
    if (op->variant == 1) {  // y_L, then the deterministic CSR gather (adds lambda x in mode 0)
      HB_TRY(launch_ax(op, op->ax_yl, 0, E, x, y, st, energy, true));
      const int64_t n = op->sz.n_owned;
      hbk::csr_gather_kernel<<<vec_grid(2 * std::max<int64_t>(n, 1)), hbk::VEC_BLOCK, 0, st>>>(
          op->csr_ptr.as<int32_t>(), op->csr_slots.as<int32_t>(), op->yL.as<double>(), x,
          op->mass_mode == 0 ? op->lam : 0.0, y, n);
      op->launches++;
      CU_TRY(cudaGetLastError());
      return HB_OK;
    }
    HB_TRY(stage_init(op, x, y, init_y, st));
    return launch_ax(op, op->ax_plain, 0, E, x, y, st, energy, true);
  }
  const int last = last_launch(op);
  cudaStream_t cs = op->comm_stream;
  auto nccl = [op](int kind, cudaStream_t c) -> int {
    if (is_ipc(op)) return ipc_exchange(op, kind, c);
    std::vector<Msg> snd, rcv;
    if (kind == 0) halo_msgs(op, snd, rcv); else assembly_msgs(op, snd, rcv);
    return nccl_exchange(op, snd, rcv, c);
  };
  HB_TRY(stage_init(op, x, y, init_y, st));
  CU_TRY(cudaEventRecord(op->ev_pack, st));
  CU_TRY(cudaStreamWaitEvent(cs, op->ev_pack, 0));
  HB_TRY(rank_phase_halo(op, x, y, st, cs, energy, last, nccl));
  return rank_phase_assembly(op, x, y, st, cs, energy, last, nccl);
}

}  // namespace

extern "C" int hb_comm_unique_id(uint8_t id[128]) {
  if (!id) { set_error("hb_comm_unique_id: null pointer"); return HB_ERR_ARG; }
  ncclUniqueId u;
  NC_TRY(ncclGetUniqueId(&u));
  static_assert(sizeof(u) == 128, "ncclUniqueId size");
  std::memcpy(id, &u, 128);
  return HB_OK;
}

extern "C" int hb_comm_create(int P, int rank, const uint8_t id[128], hb_comm** out) {
  if (!id || !out || P < 1 || rank < 0 || rank >= P) { set_error("hb_comm_create: bad argument"); return HB_ERR_ARG; }
  *out = nullptr;
  auto* c = new (std::nothrow) hb_comm();
  if (!c) { set_error("hb_comm_create: out of memory"); return HB_ERR_OOM; }
  c->P = P; c->rank = rank;
  ncclUniqueId u;
  std::memcpy(&u, id, 128);
  ncclResult_t r = ncclCommInitRank(&c->nccl, P, u, rank);
  if (r != ncclSuccess) { set_error(std::string("ncclCommInitRank: ") + ncclGetErrorString(r)); delete c; return HB_ERR_NCCL; }
  *out = c;
  return HB_OK;
}

extern "C" int hb_comm_create_ipc(int P, int rank, hb_comm** out) {
  if (!out || P < 1 || P > 32 || rank < 0 || rank >= P) { set_error("hb_comm_create_ipc: bad argument (1 <= P <= 32)"); return HB_ERR_ARG; }
  *out = nullptr;
  if (P > 1) HB_TRY(load_memops());
  auto* c = new (std::nothrow) hb_comm();
  if (!c) { set_error("hb_comm_create_ipc: out of memory"); return HB_ERR_OOM; }
  c->P = P; c->rank = rank; c->kind = 1;
  *out = c;
  return HB_OK;
}

extern "C" int hb_comm_destroy(hb_comm* c) {
  if (!c) return HB_OK;
  if (c->nccl) ncclCommDestroy(c->nccl);
  delete c;
  return HB_OK;
}

static int op_create_impl(const hb_mesh* m, hb_comm* comm, double lambda, cudaStream_t st, hb_op* op) {
  HB_TRY(hb_mesh_sizes(m, &op->sz));
  op->N = m->box.N; op->NP3 = m->NP3;
  op->mass_mode = m->box.mass_mode;
  op->lam = lambda;
  op->comm = comm;
  op->nA = m->nA; op->nH = m->nH; op->nB = m->nB;
  const int N = op->N, NP = N + 1, NP3 = m->NP3;
  const int64_t E = op->sz.E_local, NL = E * NP3, n = op->sz.n_owned;
  // constant D for this N (and the GLL weights in row 0 for the box geometry kernel)
  {
    double Dp[256] = {0};
    for (int t = 0; t < NP * NP; ++t) Dp[t] = m->D[t];
    CU_TRY(cudaMemcpyToSymbol(hbk::c_D, Dp, sizeof(Dp), sizeof(double) * 256 * N));
    // even/odd folded D and D^T for the line-owner kernel (ax_lines.cuh): rows padded to even
    // length; Me[i][m] = (M[i][m] + M[i][N-m]) / 2 (m < H), M[i][H] (middle column, odd N+1);
    // Mo[i][m] = (M[i][m] - M[i][N-m]) / 2; middle row M[H][m] (odd N+1)
    const int H = NP / 2, odd = NP & 1, HE = H + odd, HE2 = HE + (HE & 1), H2 = H + (H & 1);
    const int MAT = H * HE2 + H * H2 + H2;
    std::vector<double> eo(hbk::EO_MAX, 0.0);
    for (int tr = 0; tr < 2; ++tr) {
      auto M = [&](int i, int mm) { return tr ? m->D[mm * NP + i] : m->D[i * NP + mm]; };
      double* o = eo.data() + tr * MAT;
      for (int i = 0; i < H; ++i) {
        for (int mm = 0; mm < H; ++mm) o[i * HE2 + mm] = 0.5 * (M(i, mm) + M(i, N - mm));
        if (odd) o[i * HE2 + H] = M(i, H);
        for (int mm = 0; mm < H; ++mm) o[H * HE2 + i * H2 + mm] = 0.5 * (M(i, mm) - M(i, N - mm));
      }
      if (odd)
        for (int mm = 0; mm < H; ++mm) o[H * HE2 + H * H2 + mm] = M(H, mm);
    }
    CU_TRY(cudaMemcpyToSymbol(hbk::g_EO, eo.data(), sizeof(double) * hbk::EO_MAX, sizeof(double) * hbk::EO_MAX * N));
    CU_TRY(cudaMemcpyToSymbol(hbk::c_EO, eo.data(), sizeof(double) * hbk::eo_const(N), sizeof(double) * hbk::eo_off(N)));
  }
  // arena of everything a CG iteration re-reads besides G (candidates for L2 residency)
  {
    auto al = [](size_t b) { return (b + 255) & ~size_t(255); };
    const size_t bi = al(NL * sizeof(int32_t)), bv = al((size_t)std::max<int64_t>(n, 1) * 8);
    HB_TRY(op->arena.alloc(bi + 4 * bv));
    char* base = op->arena.as<char>();
    op->idx.view(base, NL * sizeof(int32_t));
    op->r.view(base + bi, bv);
    op->p.view(base + bi + bv, bv);
    op->Ap.view(base + bi + 2 * bv, bv);
    op->xs.view(base + bi + 3 * bv, bv);
  }
  CU_TRY(cudaMemcpyAsync(op->idx.p, m->idx.data(), NL * sizeof(int32_t), cudaMemcpyHostToDevice, st));
  HB_TRY(op->G.alloc(NL * 6 * sizeof(double)));
  if (m->has_G) {
    DevBuf tmp;
    HB_TRY(tmp.alloc(NL * 6 * sizeof(double)));
    CU_TRY(cudaMemcpyAsync(tmp.p, m->G_custom.data(), NL * 6 * sizeof(double), cudaMemcpyHostToDevice, st));
    relayout_G<<<num_sms() * 8, 256, 0, st>>>(tmp.as<double>(), op->G.as<double>(), E, NP);
    CU_TRY(cudaGetLastError());
    CU_TRY(cudaStreamSynchronize(st));
  } else if (NL > 0) {
    double wrow[256] = {0};
    for (int t = 0; t < NP; ++t) wrow[t] = m->w[t];
    CU_TRY(cudaMemcpyToSymbol(hbk::c_D, wrow, sizeof(wrow), 0));
    const double hx = m->box.ext[0], hy = m->box.ext[1], hz = m->box.ext[2];
    const double J = hx * hy * hz / 8.0;
    box_G<<<num_sms() * 8, 256, 0, st>>>(op->G.as<double>(), E, N, J * 4.0 / (hx * hx), J * 4.0 / (hy * hy), J * 4.0 / (hz * hz));
    CU_TRY(cudaGetLastError());
  }
  if (op->mass_mode == 1) {
    std::vector<double> Bh(NL);
    HB_TRY(hb_mesh_mass(m, Bh.data()));
    HB_TRY(op->B.alloc(NL * sizeof(double)));
    CU_TRY(cudaMemcpyAsync(op->B.p, Bh.data(), NL * sizeof(double), cudaMemcpyHostToDevice, st));
    CU_TRY(cudaStreamSynchronize(st));
  }
  if (m->P > 1) {
    HB_TRY(op->owned_gid.alloc(n * sizeof(int64_t)));
    CU_TRY(cudaMemcpyAsync(op->owned_gid.p, m->owned.data(), n * sizeof(int64_t), cudaMemcpyHostToDevice, st));
  }
  // CG workspace
  HB_TRY(op->partials.alloc((size_t)num_sms() * 8 * 8 + 64));
  HB_TRY(op->scal.alloc(sizeof(hbk::CgScalars)));
  CU_TRY(cudaMemsetAsync(op->scal.p, 0, sizeof(hbk::CgScalars), st));
  HB_TRY(op->dot_out.alloc(8));
  HB_TRY(op->dot_ticket.alloc(8));
  CU_TRY(cudaMemsetAsync(op->dot_ticket.p, 0, 8, st));
  CU_TRY(cudaMallocHost(&op->host_scal, sizeof(hbk::CgScalars)));
  // halo / exchange plans
  const int64_t nh = op->sz.n_halo;
  HB_TRY(op->xh.alloc(nh * 8));
  HB_TRY(op->yh.alloc(nh * 8));
  op->nbr = m->nbr;
  const size_t nn = m->nbr.size();
  op->soff.assign(nn, 0); op->scnt.assign(nn, 0); op->roff = m->recv_off; op->rcnt = m->recv_cnt;
  std::vector<int32_t> sl;
  for (size_t q = 0; q < nn; ++q) {
    op->soff[q] = (int64_t)sl.size();
    op->scnt[q] = (int64_t)m->send_loc[q].size();
    sl.insert(sl.end(), m->send_loc[q].begin(), m->send_loc[q].end());
  }
  op->n_send = (int64_t)sl.size();
  HB_TRY(op->send_loc.alloc(sl.size() * 4));
  HB_TRY(op->send_buf.alloc(sl.size() * 8));
  HB_TRY(op->recv_buf.alloc(sl.size() * 8));
  if (!sl.empty()) CU_TRY(cudaMemcpyAsync(op->send_loc.p, sl.data(), sl.size() * 4, cudaMemcpyHostToDevice, st));
  // kernels
  op->ax_plain = pick_ax(N, false, op->mass_mode == 1);
  op->ax_halo = pick_ax(N, true, op->mass_mode == 1);
  for (AxKernel* k : {&op->ax_plain, &op->ax_halo}) HB_TRY(prepare_kernel(*k));
  HB_TRY(op->e_part.alloc((size_t)std::max({op->ax_plain.grid_max, op->ax_halo.grid_max, 32 * num_sms()}) * 8 + 64));
  // P = 1: fused cooperative vector update (grid barrier instead of a second kernel)
  if (m->P == 1 && !comm) {
    int dev = 0, coop = 0, nb = 0;
    CU_TRY(cudaGetDevice(&dev));
    CU_TRY(cudaDeviceGetAttribute(&coop, cudaDevAttrCooperativeLaunch, dev));
    const char* ue = tune_env("HB_UPD_U");
    const char* me = tune_env("HB_UPD_MINB");
    // default: the batched form (first batch in flight during the p.Ap reduction) for vectors that
    // fit L2, two double2 per thread per batch at one 512-thread CTA per SM (C2: update 15.1 ->
    // 14.6 us, CG +0.7%, profiles/r2/vec/c2_update_batch.jsonl); the single-item form above that
    // (C3 N=7: the batched one is 2.7% slower; profiles/r1_update_ab.jsonl)
    const int U = ue ? atoi(ue) : (n <= 8000000 ? 2 : 0), MB = me ? atoi(me) : (U == 2 ? 1 : 2);
    auto pick = [&](auto cond) -> const void* {
      constexpr bool C = decltype(cond)::value;
      if (U == 0) return (const void*)&hbk::cg_update_fused0<C>;
      if (MB >= 2)
        return U >= 4 ? (const void*)&hbk::cg_update_fused<4, 2, C>
             : U == 2 ? (const void*)&hbk::cg_update_fused<2, 2, C> : (const void*)&hbk::cg_update_fused<1, 2, C>;
      return U >= 4 ? (const void*)&hbk::cg_update_fused<4, 1, C>
           : U == 2 ? (const void*)&hbk::cg_update_fused<2, 1, C> : (const void*)&hbk::cg_update_fused<1, 1, C>;
    };
    op->fused_fn = pick(std::false_type{});
    op->fused_fn_cond = pick(std::true_type{});
    int nb2 = 0;
    CU_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, op->fused_fn, hbk::VEC_BLOCK, 0));
    CU_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb2, op->fused_fn_cond, hbk::VEC_BLOCK, 0));
    nb = std::min(nb, nb2);
    const char* env = tune_env("HB_FUSED_UPDATE");
    if (coop && nb > 0 && !(env && env[0] == '0'))
      op->fused_grid = std::min(vec_grid(std::max<int64_t>(n, 1)), nb * num_sms());
  }
  HB_TRY(op->pp_part.alloc((size_t)std::max(op->fused_grid, 1) * 8 + 64));
  HB_TRY(op->rz_part.alloc((size_t)std::max(op->fused_grid, 1) * 8 + 64));
  {
    const char* env = tune_env("HB_PDL");
    op->pdl = op->fused_grid > 0 && !(env && env[0] == '0');
  }
  if (m->P > 1 && comm) {
    int lo, hi;
    CU_TRY(cudaDeviceGetStreamPriorityRange(&lo, &hi));
    CU_TRY(cudaStreamCreateWithPriority(&op->comm_stream, cudaStreamNonBlocking, hi));
    if (comm->kind == 1) {  // IPC mailbox (zeroed before it is exported) and pointer tables
      HB_TRY(op->mbox.alloc(mbox_bytes(m->P)));
      CU_TRY(cudaMemsetAsync(op->mbox.p, 0, mbox_bytes(m->P), st));
      HB_TRY(op->ipc_tab.alloc((size_t)2 * m->P * sizeof(void*)));
    }
  }
  CU_TRY(cudaStreamCreateWithFlags(&op->cap_stream, cudaStreamNonBlocking));
  CU_TRY(cudaStreamCreateWithFlags(&op->cap_stream2, cudaStreamNonBlocking));
  for (cudaEvent_t* e : {&op->ev_pack, &op->ev_halo, &op->ev_haloel, &op->ev_gather, &op->ev_red, &op->ev_red_done, &op->ev_cap})
    CU_TRY(cudaEventCreateWithFlags(e, cudaEventDisableTiming));
  CU_TRY(cudaStreamSynchronize(st));
  return HB_OK;
}

extern "C" int hb_op_create(const hb_mesh* m, hb_comm* comm, double lambda, void* stream, hb_op** out) {
  if (!m || !out) { set_error("hb_op_create: null pointer"); return HB_ERR_ARG; }
  *out = nullptr;
  if (m->P > 1 && comm && (comm->P != m->P || comm->rank != m->rank)) {
    set_error("hb_op_create: comm (P, rank) does not match the mesh"); return HB_ERR_STATE;
  }
  if (m->P == 1 && comm && comm->P != 1) { set_error("hb_op_create: comm given for a P=1 mesh"); return HB_ERR_STATE; }
  auto* op = new (std::nothrow) hb_op();
  if (!op) { set_error("hb_op_create: out of memory"); return HB_ERR_OOM; }
  int st = op_create_impl(m, comm, lambda, (cudaStream_t)stream, op);
  if (st != HB_OK) { delete op; return st; }
  *out = op;
  return HB_OK;
}

static int check_multi(hb_op* op, const char* fn) {
  if (op->sz.P > 1 && !op->comm) {
    set_error(std::string(fn) + ": P>1 op without a communicator (use a loopback group)");
    return HB_ERR_STATE;
  }
  if (op->sz.P > 1 && is_ipc(op) && !op->ipc_ready) {
    set_error(std::string(fn) + ": IPC op not connected (call hb_op_ipc_connect on every rank)");
    return HB_ERR_STATE;
  }
  return HB_OK;
}

// --- IPC bootstrap: export record = header + per-neighbour arrays padded to P entries
namespace {
struct IpcHeader {
  uint32_t magic, P, rank, nn;
  uint32_t has_xh, has_recv, has_send_loc, pad;
  int64_t off_p, off_Ap;  // byte offsets of p and Ap in the arena allocation (direct mode)
  cudaIpcMemHandle_t mbox, xh, recv, arena, send_loc;
};
constexpr uint32_t kIpcMagic = 0x48424950u;  // "HBIP"
size_t ipc_blob_bytes(int P) { return sizeof(IpcHeader) + (size_t)P * (4 + 4 * 8); }
}  // namespace

extern "C" int hb_op_ipc_blob_size(const hb_op* op, int64_t* bytes) {
  if (!op || !bytes) { set_error("hb_op_ipc_blob_size: null pointer"); return HB_ERR_ARG; }
  if (!is_ipc(op) || op->sz.P < 2) { set_error("hb_op_ipc_blob_size: op is not on a P>1 IPC communicator"); return HB_ERR_STATE; }
  *bytes = (int64_t)ipc_blob_bytes(op->sz.P);
  return HB_OK;
}

extern "C" int hb_op_ipc_export(const hb_op* op, uint8_t* blob) {
  if (!op || !blob) { set_error("hb_op_ipc_export: null pointer"); return HB_ERR_ARG; }
  if (!is_ipc(op) || op->sz.P < 2) { set_error("hb_op_ipc_export: op is not on a P>1 IPC communicator"); return HB_ERR_STATE; }
  const int P = op->sz.P;
  std::memset(blob, 0, ipc_blob_bytes(P));
  IpcHeader h{};
  h.magic = kIpcMagic; h.P = (uint32_t)P; h.rank = (uint32_t)op->sz.rank; h.nn = (uint32_t)op->nbr.size();
  CU_TRY(cudaIpcGetMemHandle(&h.mbox, op->mbox.p));
  h.has_xh = op->xh.p != nullptr;
  h.has_recv = op->recv_buf.p != nullptr;
  if (h.has_xh) CU_TRY(cudaIpcGetMemHandle(&h.xh, op->xh.p));
  if (h.has_recv) CU_TRY(cudaIpcGetMemHandle(&h.recv, op->recv_buf.p));
  h.has_send_loc = op->send_loc.p != nullptr;
  if (h.has_send_loc) CU_TRY(cudaIpcGetMemHandle(&h.send_loc, op->send_loc.p));
  CU_TRY(cudaIpcGetMemHandle(&h.arena, op->arena.p));
  h.off_p = op->p.as<char>() - op->arena.as<char>();
  h.off_Ap = op->Ap.as<char>() - op->arena.as<char>();
  std::memcpy(blob, &h, sizeof(h));
  int32_t* nb = reinterpret_cast<int32_t*>(blob + sizeof(h));
  int64_t* arr = reinterpret_cast<int64_t*>(blob + sizeof(h) + (size_t)P * 4);  // scnt, soff, rcnt, roff
  for (size_t i = 0; i < op->nbr.size(); ++i) {
    nb[i] = op->nbr[i];
    arr[0 * P + i] = op->scnt[i]; arr[1 * P + i] = op->soff[i];
    arr[2 * P + i] = op->rcnt[i]; arr[3 * P + i] = op->roff[i];
  }
  return HB_OK;
}

extern "C" int hb_op_set_ipc_direct(hb_op* op, int enable) {
  if (!op) { set_error("hb_op_set_ipc_direct: null pointer"); return HB_ERR_ARG; }
  if (!is_ipc(op)) { set_error("hb_op_set_ipc_direct: op is not on an IPC communicator"); return HB_ERR_STATE; }
  op->ipc_direct = enable != 0;
  return HB_OK;
}

extern "C" int hb_op_ipc_connect(hb_op* op, const uint8_t* blobs) {
  if (!op || !blobs) { set_error("hb_op_ipc_connect: null pointer"); return HB_ERR_ARG; }
  if (!is_ipc(op) || op->sz.P < 2) { set_error("hb_op_ipc_connect: op is not on a P>1 IPC communicator"); return HB_ERR_STATE; }
  if (op->ipc_ready) { set_error("hb_op_ipc_connect: already connected"); return HB_ERR_STATE; }
  const int P = op->sz.P, me = op->sz.rank;
  const size_t B = ipc_blob_bytes(P);
  op->peers.assign(P, hb_op::IpcPeer{});
  std::vector<void*> vt(2 * (size_t)P, nullptr);
  std::vector<double*> hx((size_t)op->sz.n_halo, nullptr), hy((size_t)op->sz.n_halo, nullptr);
  auto open = [op](const cudaIpcMemHandle_t& hd, void** out) -> int {
    CU_TRY(cudaIpcOpenMemHandle(out, hd, cudaIpcMemLazyEnablePeerAccess));
    op->ipc_opened.push_back(*out);
    return HB_OK;
  };
  for (int q = 0; q < P; ++q) {
    const uint8_t* b = blobs + (size_t)q * B;
    IpcHeader h;
    std::memcpy(&h, b, sizeof(h));
    if (h.magic != kIpcMagic || (int)h.P != P || (int)h.rank != q) {
      set_error("hb_op_ipc_connect: record " + std::to_string(q) + " is not rank " + std::to_string(q) + "'s export");
      return HB_ERR_STATE;
    }
    hb_op::IpcPeer& pr = op->peers[q];
    void* mb = nullptr;
    if (q == me) mb = op->mbox.p;
    else HB_TRY(open(h.mbox, &mb));
    pr.flags = static_cast<uint32_t*>(mb);
    pr.vals = reinterpret_cast<double*>(static_cast<char*>(mb) + mbox_vals_off(P));
    vt[q] = pr.vals;
    vt[P + q] = pr.flags + F_AR * P;
    if (q == me) continue;
    auto it = std::find(op->nbr.begin(), op->nbr.end(), q);
    if (it == op->nbr.end()) continue;
    const size_t i = (size_t)(it - op->nbr.begin());
    const int32_t* nb = reinterpret_cast<const int32_t*>(b + sizeof(h));
    const int64_t* arr = reinterpret_cast<const int64_t*>(b + sizeof(h) + (size_t)P * 4);
    int64_t j = -1;
    for (uint32_t t = 0; t < h.nn && t < (uint32_t)P; ++t) if (nb[t] == me) j = t;
    if (j < 0 || arr[2 * P + j] != op->scnt[i] || arr[0 * P + j] != op->rcnt[i]) {
      set_error("hb_op_ipc_connect: exchange plans of ranks " + std::to_string(me) + " and " + std::to_string(q) + " disagree");
      return HB_ERR_STATE;
    }
    if (op->scnt[i]) {  // this rank writes into q's xh
      void* p = nullptr;
      HB_TRY(open(h.xh, &p));
      pr.xh = static_cast<double*>(p);
      pr.xh_off = arr[3 * P + j];
    }
    if (op->rcnt[i]) {  // this rank writes into q's recv; direct mode reads q's p, adds into q's Ap
      void* p = nullptr;
      HB_TRY(open(h.recv, &p));
      pr.recv = static_cast<double*>(p);
      pr.recv_off = arr[1 * P + j];
      void* ar = nullptr;
      void* sl = nullptr;
      HB_TRY(open(h.arena, &ar));
      if (!h.has_send_loc) { set_error("hb_op_ipc_connect: owner without a send list"); return HB_ERR_STATE; }
      HB_TRY(open(h.send_loc, &sl));
      // q's send list for this rank is in the order of this rank's xh segment from q (gid order)
      std::vector<int32_t> loc((size_t)op->rcnt[i]);
      CU_TRY(cudaMemcpy(loc.data(), static_cast<int32_t*>(sl) + arr[1 * P + j], loc.size() * 4, cudaMemcpyDeviceToHost));
      for (size_t t = 0; t < loc.size(); ++t) {
        hx[(size_t)op->roff[i] + t] = reinterpret_cast<double*>(static_cast<char*>(ar) + h.off_p) + loc[t];
        hy[(size_t)op->roff[i] + t] = reinterpret_cast<double*>(static_cast<char*>(ar) + h.off_Ap) + loc[t];
      }
    }
  }
  for (size_t t = 0; t < hx.size(); ++t)
    if (!hx[t]) { set_error("hb_op_ipc_connect: halo node without an owner mapping"); return HB_ERR_STATE; }
  if (!hx.empty()) {
    HB_TRY(op->hx_tab.alloc(hx.size() * sizeof(double*)));
    HB_TRY(op->hy_tab.alloc(hy.size() * sizeof(double*)));
    CU_TRY(cudaMemcpy(op->hx_tab.p, hx.data(), hx.size() * sizeof(double*), cudaMemcpyHostToDevice));
    CU_TRY(cudaMemcpy(op->hy_tab.p, hy.data(), hy.size() * sizeof(double*), cudaMemcpyHostToDevice));
  }
  CU_TRY(cudaMemcpy(op->ipc_tab.p, vt.data(), vt.size() * sizeof(void*), cudaMemcpyHostToDevice));
  op->ipc_ready = true;
  return HB_OK;
}

extern "C" int hb_op_apply(hb_op* op, const double* x, double* y, void* stream) {
  if (!op || (op->sz.n_owned > 0 && (!x || !y))) { set_error("hb_op_apply: null pointer"); return HB_ERR_ARG; }
  if (x == y) { set_error("hb_op_apply: x and y must be distinct buffers"); return HB_ERR_ARG; }
  HB_TRY(check_multi(op, "hb_op_apply"));
  return apply_internal(op, x, y, true, (cudaStream_t)stream);
}

extern "C" int hb_forcing(hb_op* op, uint64_t seed, double* b, void* stream) {
  if (!op || (op->sz.n_owned > 0 && !b)) { set_error("hb_forcing: null pointer"); return HB_ERR_ARG; }
  const int64_t n = op->sz.n_owned;
  if (n == 0) return HB_OK;
  hbk::forcing_kernel<<<vec_grid(2 * n), hbk::VEC_BLOCK, 0, (cudaStream_t)stream>>>(b, op->owned_gid.as<int64_t>(), n, seed);
  op->launches++;
  CU_TRY(cudaGetLastError());
  return HB_OK;
}

static int local_dot(hb_op* op, const double* a, const double* b, cudaStream_t st) {
  const int64_t n = op->sz.n_owned;
  hbk::vec_dot<<<vec_grid(2 * std::max<int64_t>(n, 1)), hbk::VEC_BLOCK, 0, st>>>(a, b, n, op->partials.as<double>(),
                                                                               op->dot_ticket.as<uint32_t>(), op->dot_out.as<double>());
  op->launches++;
  CU_TRY(cudaGetLastError());
  return HB_OK;
}

extern "C" int hb_dot(hb_op* op, const double* a, const double* b, double* out_host, void* stream) {
  if (!op || !out_host || (op->sz.n_owned > 0 && (!a || !b))) { set_error("hb_dot: null pointer"); return HB_ERR_ARG; }
  HB_TRY(check_multi(op, "hb_dot"));
  cudaStream_t st = (cudaStream_t)stream;
  HB_TRY(local_dot(op, a, b, st));
  HB_TRY(allreduce_sum(op, op->dot_out.as<double>(), st));
  CU_TRY(cudaMemcpyAsync(out_host, op->dot_out.p, 8, cudaMemcpyDeviceToHost, st));
  CU_TRY(cudaStreamSynchronize(st));
  return HB_OK;
}

namespace {

double lam_init(const hb_op* op) { return op->mass_mode == 0 ? op->lam : 0.0; }
double lam_pp(const hb_op* op) { return op->mass_mode == 0 ? op->lam : 0.0; }

int cg_init(hb_op* op, const double* b, double* x, cudaStream_t st) {
  const int64_t n = op->sz.n_owned;
  const bool fused = op->fused_grid > 0;
  hbk::cg_init<<<fused ? op->fused_grid : vec_grid(2 * std::max<int64_t>(n, 1)), hbk::VEC_BLOCK, 0, st>>>(
      b, x, op->r.as<double>(), op->p.as<double>(), op->Ap.as<double>(), n, lam_init(op),
      op->partials.as<double>(), op->scal.as<hbk::CgScalars>(), fused ? op->pp_part.as<double>() : nullptr,
      op->jacobi ? op->invd.as<double>() : nullptr);
  op->launches++;
  CU_TRY(cudaGetLastError());
  hbk::CgScalars* s = op->scal.as<hbk::CgScalars>();
  HB_TRY(allreduce_sum(op, &s->rr_new, st));
  if (direct_mode(op)) HB_TRY(ipc_signal_ready(op, st));  // p = b and Ap = lambda p are written
  return HB_OK;
}

// One CG iteration after the operator (which published p.Ap): x/r update + r.r, then p update.
int cg_vec_part1(hb_op* op, double* x, cudaStream_t st) {
  const int64_t n = op->sz.n_owned;
  hbk::CgScalars* s = op->scal.as<hbk::CgScalars>();
  const int gv = vec_grid(std::max<int64_t>(n, 1));
  HB_TRY(allreduce_sum(op, &s->pAp, st));
  if (op->fused_grid > 0) {  // one GPU: the whole vector part of the iteration, one cooperative kernel
    HB_TRY(phase_event(op, op->t_xr, true, st));
    double* xp = x;
    double* pp = op->p.as<double>();
    double* rp = op->r.as<double>();
    double* ap = op->Ap.as<double>();
    int64_t nn = n;
    const double* ep = op->e_part.as<double>();
    int nep = op->last_grid;
    double* ppp = op->pp_part.as<double>();
    double lpp = lam_pp(op), li = lam_init(op);
    double* rrp = op->partials.as<double>();
    double* hp = op->hist.as<double>();
    const double* ivd = op->jacobi ? op->invd.as<double>() : nullptr;
    double* rzp = op->rz_part.as<double>();
    hbk::CondTest ct = op->cond_test;
    void* args[] = {&xp, &pp, &rp, &ap, &nn, &ep, &nep, &ppp, &lpp, &li, &rrp, &s, &hp, &ivd, &rzp, &ct};
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(op->fused_grid); cfg.blockDim = dim3(hbk::VEC_BLOCK); cfg.stream = st;
    cudaLaunchAttribute at[2];
    at[0].id = cudaLaunchAttributeCooperative;
    at[0].val.cooperative = 1;
    at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[1].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at; cfg.numAttrs = op->pdl ? 2 : 1;
    CU_TRY(cudaLaunchKernelExC(&cfg, ct.on ? op->fused_fn_cond : op->fused_fn, args));
    op->launches++;
    return phase_event(op, op->t_xr, false, st);
  }
  if (!op->comm || op->comm->P == 1) {  // one GPU: energy reduction + x and r updates in one pass
    HB_TRY(phase_event(op, op->t_xr, true, st));
    hbk::cg_update_xr_e<<<gv, hbk::VEC_BLOCK, 0, st>>>(x, op->p.as<double>(), op->r.as<double>(), op->Ap.as<double>(),
                                                       n, op->e_part.as<double>(), op->last_grid, lam_pp(op),
                                                       op->partials.as<double>(), s, op->hist.as<double>());
    op->launches++;
    CU_TRY(cudaGetLastError());
    return phase_event(op, op->t_xr, false, st);
  }
  // P > 1: r update + r.r, then the r.r allreduce on the comm stream overlapped with
  // the x AXPY on the compute stream
  hbk::cg_update_r<<<gv, hbk::VEC_BLOCK, 0, st>>>(op->r.as<double>(), op->Ap.as<double>(), n,
                                                  op->partials.as<double>(), s);
  op->launches++;
  CU_TRY(cudaEventRecord(op->ev_red, st));
  CU_TRY(cudaStreamWaitEvent(op->comm_stream, op->ev_red, 0));
  HB_TRY(allreduce_sum(op, &s->rr_loc, op->comm_stream));
  CU_TRY(cudaEventRecord(op->ev_red_done, op->comm_stream));
  hbk::cg_update_x<<<gv, hbk::VEC_BLOCK, 0, st>>>(x, op->p.as<double>(), n, s);
  op->launches++;
  CU_TRY(cudaStreamWaitEvent(st, op->ev_red_done, 0));
  CU_TRY(cudaGetLastError());
  return HB_OK;
}

int cg_vec_part2(hb_op* op, cudaStream_t st) {
  const int64_t n = op->sz.n_owned;
  if (op->fused_grid > 0) {  // done inside cg_update_fused
    op->last_timed = false;
    return HB_OK;
  }
  HB_TRY(phase_event(op, op->t_p, true, st));
  hbk::cg_update_p<<<vec_grid(std::max<int64_t>(n, 1)), hbk::VEC_BLOCK, 0, st>>>(
      op->p.as<double>(), op->r.as<double>(), op->Ap.as<double>(), n, lam_init(op), op->partials.as<double>(),
      op->scal.as<hbk::CgScalars>(), op->tol_eps, op->tol_max);
  op->launches++;
  CU_TRY(cudaGetLastError());
  HB_TRY(phase_event(op, op->t_p, false, st));
  op->last_timed = false;
  return HB_OK;
}

int cg_iteration(hb_op* op, double* x, cudaStream_t st) {
  if (direct_mode(op)) {
    HB_TRY(direct_apply(op, st));
    HB_TRY(cg_vec_part1(op, x, st));
    HB_TRY(cg_vec_part2(op, st));
    return ipc_signal_ready(op, st);
  }
  if (!op->timing_vec_only) HB_TRY(apply_internal(op, op->p.as<double>(), op->Ap.as<double>(), false, st, true));
  HB_TRY(cg_vec_part1(op, x, st));
  return cg_vec_part2(op, st);
}

int ensure_hist(hb_op* op, int32_t K) {
  size_t need = (size_t)(K + 1) * 8;
  if (op->hist.bytes < need) {
    // graphs reference the old history buffer
    for (auto& kv : op->graphs) cudaGraphExecDestroy(kv.second.exec);
    op->graphs.clear();
    for (auto& kv : op->tol_graphs) cudaGraphExecDestroy(kv.second.exec);
    op->tol_graphs.clear();
    for (auto& kv : op->chunk_graphs) cudaGraphExecDestroy(kv.second.exec);
    op->chunk_graphs.clear();
    for (auto& kv : op->scat_graphs) cudaGraphExecDestroy(kv.second.exec);
    op->scat_graphs.clear();
    HB_TRY(op->hist.alloc(need));
  }
  return HB_OK;
}

int finish_result(hb_op* op, int32_t iters, double* rr_hist_host, hb_cg_result* res, cudaStream_t st) {
  CU_TRY(cudaMemcpyAsync(op->host_scal, op->scal.p, sizeof(hbk::CgScalars), cudaMemcpyDeviceToHost, st));
  if (rr_hist_host && iters > 0)
    CU_TRY(cudaMemcpyAsync(rr_hist_host, op->hist.p, (size_t)iters * 8, cudaMemcpyDeviceToHost, st));
  CU_TRY(cudaStreamSynchronize(st));
  const hbk::CgScalars* hs = reinterpret_cast<const hbk::CgScalars*>(op->host_scal);
  if (rr_hist_host) rr_hist_host[iters] = hs->rr_new;
  if (res) {
    res->iterations = iters;
    res->rr_final = hs->rr_new;
    res->rr0 = rr_hist_host ? rr_hist_host[0] : (iters == 0 ? hs->rr_new : NAN);
  }
  return HB_OK;
}

int cg_fixed(hb_op* op, const double* b, double* x, int32_t K, double* rr_hist_host, hb_cg_result* res,
             cudaStream_t st) {
  HB_TRY(ensure_hist(op, K));
  auto stream_loop = [&]() -> int {  // stream-ordered loop, no graph
    if (op->profiling) { op->prof_used = 0; op->prof_seq = 0; op->t_xr.used = 0; op->t_p.used = 0; }
    HB_TRY(cg_init(op, b, x, st));
    for (int32_t j = 0; j < K; ++j) HB_TRY(cg_iteration(op, x, st));
    return finish_result(op, K, rr_hist_host, res, st);
  };
  // IPC: the transport's flags carry per-call sequence numbers, so a replayed graph would repeat
  // stale values; NCCL: graph capture is the default, the stream loop the fallback if capturing
  // the communicator's calls fails on this system
  if (is_ipc(op) || !op->graph_ok) return stream_loop();
  hb_op::GraphKey key{K, b, x, op->profiling, op->timing_vec_only, st};
  auto it = op->graphs.find(key);
  if (op->profiling) { op->prof_used = 0; op->prof_seq = 0; op->t_xr.used = 0; op->t_p.used = 0; }  // a profiling graph records into events 0..n-1
  if (it == op->graphs.end()) {
    int64_t l0 = op->launches;
    cudaGraph_t graph = nullptr;
    cudaStream_t cs = op->cap_stream;
    CU_TRY(cudaStreamBeginCapture(cs, cudaStreamCaptureModeThreadLocal));
    int status = cg_init(op, b, x, cs);
    for (int32_t j = 0; j < K && status == HB_OK; ++j) status = cg_iteration(op, x, cs);
    cudaError_t ce = cudaStreamEndCapture(cs, &graph);
    cudaGraphExec_t exec = nullptr;
    cudaError_t ie = cudaErrorUnknown;
    if (status == HB_OK && ce == cudaSuccess) ie = cudaGraphInstantiate(&exec, graph, 0);
    if (ce == cudaSuccess && graph) cudaGraphDestroy(graph);
    if (status != HB_OK || ce != cudaSuccess || ie != cudaSuccess) {
      op->launches = l0;
      if (op->comm && op->comm->P > 1) {  // NCCL calls could not be captured: run uncaptured from now on
        (void)cudaGetLastError();
        op->graph_ok = false;
        return stream_loop();
      }
      if (status != HB_OK) return status;
      CU_TRY(ce);
      CU_TRY(ie);
    }
    it = op->graphs.emplace(key, hb_op::GraphVal{exec, op->launches - l0, op->prof_used, op->t_xr.used, op->t_p.used}).first;
    op->launches = l0;
  }
  op->prof_used = it->second.prof_events;
  op->t_xr.used = it->second.prof_xr;
  op->t_p.used = it->second.prof_p;
  CU_TRY(cudaGraphLaunch(it->second.exec, st));
  op->launches += it->second.launches;
  return finish_result(op, K, rr_hist_host, res, st);
}

// Tolerance mode fully on the device (P = 1): one CUDA graph
//   init -> cg_continue(first) -> WHILE(cond) { operator ; fused vector update ; cg_continue }
// captured once per (K, b, x, eps) and replayed; the host synchronises only at the end.
int cg_tol_graph(hb_op* op, const double* b, double* x, int32_t max_iters, double eps, double* rr_hist_host,
                 hb_cg_result* res, cudaStream_t st) {
  HB_TRY(ensure_hist(op, max_iters));
  hb_op::TolKey key{max_iters, b, x, eps, st};
  auto it = op->tol_graphs.find(key);
  if (op->profiling) { op->prof_used = 0; op->prof_seq = 0; op->t_xr.used = 0; op->t_p.used = 0; }
  if (it == op->tol_graphs.end()) {
    const int64_t l0 = op->launches;
    const bool prof = op->profiling;
    op->profiling = false;  // a data-dependent trip count cannot own a fixed event set
    cudaStream_t cs = op->cap_stream, cs2 = op->cap_stream2;
    hbk::CgScalars* s = op->scal.as<hbk::CgScalars>();
    cudaGraph_t graph = nullptr;
    int status = HB_OK;
    auto fail = [&](cudaError_t e, const char* what) {
      if (e != cudaSuccess && status == HB_OK) {
        (void)cudaGetLastError();
        set_error(std::string("cg_tol_graph: ") + what + ": " + cudaGetErrorString(e));
        status = HB_ERR_CUDA;
      }
    };
    fail(cudaStreamBeginCapture(cs, cudaStreamCaptureModeThreadLocal), "begin capture");
    if (status == HB_OK) status = cg_init(op, b, x, cs);
    cudaGraphConditionalHandle h = 0;
    cudaGraph_t cap_graph = nullptr;
    const cudaGraphNode_t* deps = nullptr;
    size_t ndeps = 0;
    cudaStreamCaptureStatus cst;
    if (status == HB_OK) fail(cudaStreamGetCaptureInfo(cs, &cst, nullptr, &cap_graph, &deps, &ndeps), "capture info");
    if (status == HB_OK) fail(cudaGraphConditionalHandleCreate(&h, cap_graph, 0, 0), "conditional handle");
    if (status == HB_OK) {
      hbk::cg_continue<<<1, 1, 0, cs>>>(h, s, eps, max_iters, 1);
      fail(cudaGetLastError(), "cg_continue");
    }
    cudaGraphNode_t cond = nullptr;
    cudaGraph_t body = nullptr;
    if (status == HB_OK) fail(cudaStreamGetCaptureInfo(cs, &cst, nullptr, &cap_graph, &deps, &ndeps), "capture info");
    if (status == HB_OK) {
      cudaGraphNodeParams cp = {};
      cp.type = cudaGraphNodeTypeConditional;
      cp.conditional.handle = h;
      cp.conditional.type = cudaGraphCondTypeWhile;
      cp.conditional.size = 1;
      fail(cudaGraphAddNode(&cond, cap_graph, deps, ndeps, &cp), "add WHILE node");
      if (status == HB_OK) body = cp.conditional.phGraph_out[0];
    }
    if (status == HB_OK) fail(cudaStreamUpdateCaptureDependencies(cs, &cond, 1, cudaStreamSetCaptureDependencies),
                              "update capture deps");
    if (status == HB_OK) {  // loop body on a second stream captured into the WHILE node's graph
      fail(cudaStreamBeginCaptureToGraph(cs2, body, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal),
           "begin body capture");
      if (status == HB_OK) {
        // with the fused vector update the loop test runs inside it (no separate kernel)
        const bool folded = op->fused_grid > 0;
        if (folded) op->cond_test = hbk::CondTest{h, eps, max_iters, 1};
        status = cg_iteration(op, x, cs2);
        op->cond_test.on = 0;
        if (status == HB_OK && !folded) {
          hbk::cg_continue<<<1, 1, 0, cs2>>>(h, s, eps, max_iters, 0);
          fail(cudaGetLastError(), "cg_continue");
        }
        cudaGraph_t bg = nullptr;
        fail(cudaStreamEndCapture(cs2, &bg), "end body capture");
      }
    }
    cudaError_t ce = cudaStreamEndCapture(cs, &graph);
    op->profiling = prof;
    if (status != HB_OK) { if (ce == cudaSuccess && graph) cudaGraphDestroy(graph); return status; }
    CU_TRY(ce);
    cudaGraphExec_t exec;
    cudaError_t ie = cudaGraphInstantiate(&exec, graph, 0);
    cudaGraphDestroy(graph);
    CU_TRY(ie);
    it = op->tol_graphs.emplace(key, hb_op::GraphVal{exec, op->launches - l0, 0, 0, 0}).first;
    op->launches = l0;
  }
  CU_TRY(cudaGraphLaunch(it->second.exec, st));
  CU_TRY(cudaMemcpyAsync(op->host_scal, op->scal.p, sizeof(hbk::CgScalars), cudaMemcpyDeviceToHost, st));
  CU_TRY(cudaStreamSynchronize(st));
  const hbk::CgScalars* hs = reinterpret_cast<const hbk::CgScalars*>(op->host_scal);
  const int32_t iters = hs->it;
  op->launches += 1 + (int64_t)iters * (op->fused_grid > 0 ? 2 : 3);  // init + (operator, update[, loop test]) per trip
  if (hs->flags & 1) {
    set_error("hb_cg_solve: breakdown (p.Ap <= 0 or non-finite) at iteration " + std::to_string(iters - 1));
    return HB_ERR_BREAKDOWN;
  }
  return finish_result(op, iters, rr_hist_host, res, st);
}

int cg_tol(hb_op* op, const double* b, double* x, int32_t max_iters, double eps, double* rr_hist_host,
           hb_cg_result* res, cudaStream_t st) {
  HB_TRY(ensure_hist(op, max_iters));
  hbk::CgScalars* hs = reinterpret_cast<hbk::CgScalars*>(op->host_scal);
  HB_TRY(cg_init(op, b, x, st));
  CU_TRY(cudaMemcpyAsync(op->host_scal, op->scal.p, sizeof(hbk::CgScalars), cudaMemcpyDeviceToHost, st));
  CU_TRY(cudaStreamSynchronize(st));
  int32_t j = 0;
  double rr = hs->rr_new;
  while (j < max_iters && rr > eps) {
    if (direct_mode(op)) HB_TRY(direct_apply(op, st));
    else HB_TRY(apply_internal(op, op->p.as<double>(), op->Ap.as<double>(), false, st, true));
    HB_TRY(cg_vec_part1(op, x, st));
    CU_TRY(cudaMemcpyAsync(op->host_scal, op->scal.p, sizeof(hbk::CgScalars), cudaMemcpyDeviceToHost, st));
    CU_TRY(cudaStreamSynchronize(st));
    if (!(hs->pAp > 0.0) || !std::isfinite(hs->pAp) || !std::isfinite(hs->rr_loc)) {
      set_error("hb_cg_solve: breakdown (p.Ap <= 0 or non-finite) at iteration " + std::to_string(j));
      return HB_ERR_BREAKDOWN;
    }
    HB_TRY(cg_vec_part2(op, st));
    if (direct_mode(op)) HB_TRY(ipc_signal_ready(op, st));
    ++j;
    rr = hs->rr_loc;
  }
  return finish_result(op, j, rr_hist_host, res, st);
}

// Tolerance mode with P > 1 without a host round trip per iteration: iterations are enqueued in
// chunks of kTolChunk; cg_update_p takes the loop test on the device (global r.r, so every rank
// decides alike) and, once the solve has finished, the remaining iterations of the chunk are
// no-ops (every iteration kernel returns at once; the exchanges and allreduces still run, on
// values nobody reads: r.r goes through rr_loc, so rr_new is not re-summed).  The host reads the
// scalars once per chunk.  NCCL: each chunk is one captured graph, replayed; IPC: stream-ordered
// (its flags carry per-call sequence numbers).
constexpr int32_t kTolChunk = 8;

int cg_tol_chunked(hb_op* op, const double* b, double* x, int32_t max_iters, double eps, double* rr_hist_host,
                   hb_cg_result* res, cudaStream_t st) {
  HB_TRY(ensure_hist(op, max_iters + kTolChunk));
  hbk::CgScalars* hs = reinterpret_cast<hbk::CgScalars*>(op->host_scal);
  if (op->profiling) { op->prof_used = 0; op->prof_seq = 0; op->t_xr.used = 0; op->t_p.used = 0; }
  HB_TRY(cg_init(op, b, x, st));
  CU_TRY(cudaMemcpyAsync(op->host_scal, op->scal.p, sizeof(hbk::CgScalars), cudaMemcpyDeviceToHost, st));
  CU_TRY(cudaStreamSynchronize(st));
  if (!(hs->rr_new > eps) || max_iters == 0) return finish_result(op, 0, rr_hist_host, res, st);
  struct Restore {
    hb_op* o;
    ~Restore() { o->tol_eps = -1.0; o->tol_max = INT32_MAX; }
  } restore{op};
  op->tol_eps = eps;
  op->tol_max = max_iters;
  cudaGraphExec_t exec = nullptr;
  int64_t exec_launches = 0;
  if (!is_ipc(op) && op->graph_ok) {  // one graph per (max_iters, b, x, eps): kTolChunk predicated iterations
    hb_op::TolKey key{max_iters, b, x, eps, st};
    auto it = op->chunk_graphs.find(key);
    if (it == op->chunk_graphs.end()) {
      const int64_t l0 = op->launches;
      const bool prof = op->profiling;
      op->profiling = false;
      cudaGraph_t graph = nullptr;
      cudaStream_t cs = op->cap_stream;
      CU_TRY(cudaStreamBeginCapture(cs, cudaStreamCaptureModeThreadLocal));
      int status = HB_OK;
      for (int32_t j = 0; j < kTolChunk && status == HB_OK; ++j) status = cg_iteration(op, x, cs);
      cudaError_t ce = cudaStreamEndCapture(cs, &graph);
      op->profiling = prof;
      cudaGraphExec_t ex = nullptr;
      cudaError_t ie = cudaErrorUnknown;
      if (status == HB_OK && ce == cudaSuccess) ie = cudaGraphInstantiate(&ex, graph, 0);
      if (ce == cudaSuccess && graph) cudaGraphDestroy(graph);
      const int64_t captured = op->launches - l0;
      op->launches = l0;
      if (status == HB_OK && ce == cudaSuccess && ie == cudaSuccess) {
        it = op->chunk_graphs.emplace(key, hb_op::GraphVal{ex, captured, 0, 0, 0}).first;
      } else {  // the communicator's calls could not be captured: stream-ordered chunks
        (void)cudaGetLastError();
        op->graph_ok = false;
      }
    }
    if (op->graph_ok) {
      exec = it->second.exec;
      exec_launches = it->second.launches;
    }
  }
  for (int32_t launched = 0; launched < max_iters; launched += kTolChunk) {
    if (exec) {
      CU_TRY(cudaGraphLaunch(exec, st));
      op->launches += exec_launches;
    } else {
      for (int32_t j = 0; j < kTolChunk; ++j) HB_TRY(cg_iteration(op, x, st));
    }
    CU_TRY(cudaMemcpyAsync(op->host_scal, op->scal.p, sizeof(hbk::CgScalars), cudaMemcpyDeviceToHost, st));
    CU_TRY(cudaStreamSynchronize(st));
    if (hs->flags & 2) break;
  }
  if (hs->flags & 1) {
    set_error("hb_cg_solve: breakdown (p.Ap <= 0 or non-finite) at iteration " + std::to_string(hs->it));
    return HB_ERR_BREAKDOWN;
  }
  return finish_result(op, hs->it, rr_hist_host, res, st);
}

}  // namespace

extern "C" int hb_cg_solve(hb_op* op, const double* b, double* x, int32_t max_iters, double eps,
                           double* rr_hist_host, hb_cg_result* res, void* stream) {
  if (!op || (op->sz.n_owned > 0 && (!b || !x))) { set_error("hb_cg_solve: null pointer"); return HB_ERR_ARG; }
  if (max_iters < 0) { set_error("hb_cg_solve: max_iters must be >= 0"); return HB_ERR_ARG; }
  HB_TRY(check_multi(op, "hb_cg_solve"));
  cudaStream_t st = (cudaStream_t)stream;
  if (eps < 0) return cg_fixed(op, b, x, max_iters, rr_hist_host, res, st);
  if (op->fused_grid > 0 && op->tol_device_loop) return cg_tol_graph(op, b, x, max_iters, eps, rr_hist_host, res, st);
  if (op->comm && op->comm->P > 1 && op->tol_device_loop)
    return cg_tol_chunked(op, b, x, max_iters, eps, rr_hist_host, res, st);
  return cg_tol(op, b, x, max_iters, eps, rr_hist_host, res, st);
}

extern "C" int hb_cg_solve_host(hb_op* op, const double* b_host, double* x_host, int32_t max_iters, double eps,
                                double* rr_hist_host, hb_cg_result* res, void* stream) {
  if (!op || (op->sz.n_owned > 0 && (!b_host || !x_host))) { set_error("hb_cg_solve_host: null pointer"); return HB_ERR_ARG; }
  cudaStream_t st = (cudaStream_t)stream;
  const size_t bytes = (size_t)op->sz.n_owned * 8;
  // b is staged through the internal x buffer's twin: use r as the device copy of b
  // (cg_init reads b before writing r, element by element, so aliasing is safe).
  double* b_dev = op->r.as<double>();
  if (bytes) CU_TRY(cudaMemcpyAsync(b_dev, b_host, bytes, cudaMemcpyHostToDevice, st));
  HB_TRY(hb_cg_solve(op, b_dev, op->xs.as<double>(), max_iters, eps, rr_hist_host, res, stream));
  if (bytes) CU_TRY(cudaMemcpyAsync(x_host, op->xs.p, bytes, cudaMemcpyDeviceToHost, st));
  CU_TRY(cudaStreamSynchronize(st));
  return HB_OK;
}

// CSR of Z^T over owned DOFs, slots in ascending (e, n) order (counting sort by gid), and the
// y_L buffer -- shared by the deterministic variant and the scattered-storage CG
static int ensure_csr(hb_op* op) {
  if (op->yL.p) return HB_OK;
  const int64_t n = op->sz.n_owned, NL = op->sz.N_L;
  std::vector<int32_t> idx(NL);
  CU_TRY(cudaMemcpy(idx.data(), op->idx.p, NL * 4, cudaMemcpyDeviceToHost));
  std::vector<int32_t> ptr(n + 1, 0), slots(NL);
  for (int64_t t = 0; t < NL; ++t) ptr[idx[t] + 1]++;
  for (int64_t g = 0; g < n; ++g) ptr[g + 1] += ptr[g];
  std::vector<int32_t> fill(ptr.begin(), ptr.end() - 1);
  for (int64_t t = 0; t < NL; ++t) slots[fill[idx[t]]++] = (int32_t)t;
  HB_TRY(op->csr_ptr.alloc((n + 1) * 4));
  HB_TRY(op->csr_slots.alloc(NL * 4));
  HB_TRY(op->yL.alloc(NL * 8));
  CU_TRY(cudaMemcpy(op->csr_ptr.p, ptr.data(), (n + 1) * 4, cudaMemcpyHostToDevice));
  CU_TRY(cudaMemcpy(op->csr_slots.p, slots.data(), NL * 4, cudaMemcpyHostToDevice));
  return HB_OK;
}

extern "C" int hb_op_set_variant(hb_op* op, int variant, void* stream) {
  if (!op || variant < 0 || variant > 1) { set_error("hb_op_set_variant: bad argument"); return HB_ERR_ARG; }
  if (variant >= 1 && (op->sz.P > 1 || op->comm)) {
    set_error("hb_op_set_variant: variant 1 is available for P = 1 only");
    return HB_ERR_STATE;
  }
  cudaStream_t st = (cudaStream_t)stream;
  if (variant == 1) {
    HB_TRY(ensure_csr(op));
    if (!op->ax_yl.fn) {
      op->ax_yl = pick_ax(op->N, false, op->mass_mode == 1, 1);
      HB_TRY(prepare_kernel(op->ax_yl));
    }
  }
  (void)st;
  if (variant != op->variant) {
    for (auto& kv : op->graphs) cudaGraphExecDestroy(kv.second.exec);
    op->graphs.clear();
    for (auto& kv : op->tol_graphs) cudaGraphExecDestroy(kv.second.exec);
    op->tol_graphs.clear();
    for (auto& kv : op->chunk_graphs) cudaGraphExecDestroy(kv.second.exec);
    op->chunk_graphs.clear();
  }
  op->variant = variant;
  return HB_OK;
}

// ---------------------------------------------------------------- scattered storage CG
namespace {
int scat_setup(hb_op* op) {
  HB_TRY(ensure_csr(op));
  if (!op->ax_scat.fn) {
    op->ax_scat = pick_ax(op->N, false, false, 2);
    HB_TRY(prepare_kernel(op->ax_scat));
  }
  if (op->sW.p) return HB_OK;
  const int64_t NL = op->sz.N_L;
  for (DevBuf* b : {&op->sL_x, &op->sL_r, &op->sL_p, &op->sL_w, &op->sW}) HB_TRY(b->alloc(NL * 8));
  // W_s = 1 / (number of slots of the slot's DOF): from the CSR row lengths
  const int64_t n = op->sz.n_owned;
  std::vector<int32_t> ptr(n + 1), idx(NL);
  CU_TRY(cudaMemcpy(ptr.data(), op->csr_ptr.p, (n + 1) * 4, cudaMemcpyDeviceToHost));
  CU_TRY(cudaMemcpy(idx.data(), op->idx.p, NL * 4, cudaMemcpyDeviceToHost));
  std::vector<double> W(NL);
  for (int64_t t = 0; t < NL; ++t) W[t] = 1.0 / (double)(ptr[idx[t] + 1] - ptr[idx[t]]);
  CU_TRY(cudaMemcpy(op->sW.p, W.data(), NL * 8, cudaMemcpyHostToDevice));
  return HB_OK;
}

int scat_iteration(hb_op* op, cudaStream_t st) {
  const int64_t n = op->sz.n_owned, NL = op->sz.N_L;
  hbk::CgScalars* s = op->scal.as<hbk::CgScalars>();
  const int gl = vec_grid(2 * NL);
  op->scat_mode = true;
  const int stt = launch_ax(op, op->ax_scat, 0, op->sz.E_local, nullptr, nullptr, st);  // y_L = S_L p_L
  op->scat_mode = false;
  HB_TRY(stt);
  hbk::gs_scatter_kernel<<<vec_grid(2 * n), hbk::VEC_BLOCK, 0, st>>>(op->csr_ptr.as<int32_t>(), op->csr_slots.as<int32_t>(),
                                                                   op->yL.as<double>(), op->sL_p.as<double>(), op->lam,
                                                                   op->sL_w.as<double>(), n);
  hbk::wdot_kernel<<<gl, hbk::VEC_BLOCK, 0, st>>>(op->sW.as<double>(), op->sL_p.as<double>(), op->sL_w.as<double>(), NL,
                                                  op->partials.as<double>(), &s->ticket, &s->pAp);
  hbk::scat_update_xr<<<gl, hbk::VEC_BLOCK, 0, st>>>(op->sL_x.as<double>(), op->sL_p.as<double>(), op->sL_r.as<double>(),
                                                     op->sL_w.as<double>(), op->sW.as<double>(), NL,
                                                     op->partials.as<double>(), s, op->hist.as<double>());
  hbk::scat_update_p<<<gl, hbk::VEC_BLOCK, 0, st>>>(op->sL_p.as<double>(), op->sL_r.as<double>(), NL, s);
  op->launches += 4;
  CU_TRY(cudaGetLastError());
  return HB_OK;
}

int scat_init(hb_op* op, const double* b, cudaStream_t st) {
  const int64_t NL = op->sz.N_L;
  hbk::CgScalars* s = op->scal.as<hbk::CgScalars>();
  const int gl = vec_grid(2 * NL);
  hbk::scatter_kernel<<<gl, hbk::VEC_BLOCK, 0, st>>>(op->idx.as<int32_t>(), b, op->sL_r.as<double>(), NL);
  CU_TRY(cudaMemcpyAsync(op->sL_p.p, op->sL_r.p, NL * 8, cudaMemcpyDeviceToDevice, st));
  CU_TRY(cudaMemsetAsync(op->sL_x.p, 0, NL * 8, st));
  CU_TRY(cudaMemsetAsync(&s->it, 0, sizeof(int32_t), st));
  hbk::wdot_kernel<<<gl, hbk::VEC_BLOCK, 0, st>>>(op->sW.as<double>(), op->sL_r.as<double>(), op->sL_r.as<double>(), NL,
                                                  op->partials.as<double>(), &s->ticket, &s->rr_new);
  op->launches += 2;
  CU_TRY(cudaGetLastError());
  return HB_OK;
}
}  // namespace

extern "C" int hb_cg_solve_scattered(hb_op* op, const double* b, double* x, int32_t max_iters, double eps,
                                     double* rr_hist_host, hb_cg_result* res, void* stream) {
  if (!op || (op->sz.n_owned > 0 && (!b || !x)) || max_iters < 0) { set_error("hb_cg_solve_scattered: bad argument"); return HB_ERR_ARG; }
  if (op->sz.P > 1 || op->comm || op->mass_mode != 0) {
    set_error("hb_cg_solve_scattered: NekBone's scattered storage is implemented for P = 1, mass mode 0");
    return HB_ERR_STATE;
  }
  cudaStream_t st = (cudaStream_t)stream;
  HB_TRY(scat_setup(op));
  HB_TRY(ensure_hist(op, max_iters));
  int32_t iters = 0;
  if (eps < 0) {  // fixed mode: one captured graph per (K, b, x), like hb_cg_solve
    auto key = std::make_tuple(max_iters, b, x);
    auto it = op->scat_graphs.find(key);
    if (it == op->scat_graphs.end()) {
      const int64_t l0 = op->launches;
      cudaStream_t cs = op->cap_stream;
      cudaGraph_t graph;
      CU_TRY(cudaStreamBeginCapture(cs, cudaStreamCaptureModeThreadLocal));
      int status = scat_init(op, b, cs);
      for (int32_t j = 0; j < max_iters && status == HB_OK; ++j) status = scat_iteration(op, cs);
      cudaError_t ce = cudaStreamEndCapture(cs, &graph);
      if (status != HB_OK) { if (ce == cudaSuccess) cudaGraphDestroy(graph); return status; }
      CU_TRY(ce);
      cudaGraphExec_t exec;
      cudaError_t ie = cudaGraphInstantiate(&exec, graph, 0);
      cudaGraphDestroy(graph);
      CU_TRY(ie);
      it = op->scat_graphs.emplace(key, hb_op::GraphVal{exec, op->launches - l0, 0, 0, 0}).first;
      op->launches = l0;
    }
    CU_TRY(cudaGraphLaunch(it->second.exec, st));
    op->launches += it->second.launches;
    iters = max_iters;
  } else {
    HB_TRY(scat_init(op, b, st));
    hbk::CgScalars* hs = reinterpret_cast<hbk::CgScalars*>(op->host_scal);
    CU_TRY(cudaMemcpyAsync(op->host_scal, op->scal.p, sizeof(hbk::CgScalars), cudaMemcpyDeviceToHost, st));
    CU_TRY(cudaStreamSynchronize(st));
    while (iters < max_iters && hs->rr_new > eps) {
      HB_TRY(scat_iteration(op, st));
      CU_TRY(cudaMemcpyAsync(op->host_scal, op->scal.p, sizeof(hbk::CgScalars), cudaMemcpyDeviceToHost, st));
      CU_TRY(cudaStreamSynchronize(st));
      if (!(hs->pAp > 0.0) || !std::isfinite(hs->pAp)) {
        set_error("hb_cg_solve_scattered: breakdown at iteration " + std::to_string(iters));
        return HB_ERR_BREAKDOWN;
      }
      ++iters;
    }
  }
  const int64_t n = op->sz.n_owned;
  hbk::pick_kernel<<<vec_grid(2 * n), hbk::VEC_BLOCK, 0, st>>>(op->csr_ptr.as<int32_t>(), op->csr_slots.as<int32_t>(),
                                                             op->sL_x.as<double>(), x, n);
  op->launches++;
  CU_TRY(cudaGetLastError());
  return finish_result(op, iters, rr_hist_host, res, st);
}

extern "C" int hb_op_set_jacobi(hb_op* op, int enable, void* stream) {
  if (!op) { set_error("hb_op_set_jacobi: null pointer"); return HB_ERR_ARG; }
  if (enable && op->fused_grid <= 0) {
    set_error("hb_op_set_jacobi: the Jacobi-preconditioned CG is available for P = 1 only");
    return HB_ERR_STATE;
  }
  cudaStream_t st = (cudaStream_t)stream;
  if (enable && !op->invd.p) {
    const int64_t n = op->sz.n_owned, E = op->sz.E_local;
    HB_TRY(op->invd.alloc((size_t)std::max<int64_t>(n, 1) * 8));
    CU_TRY(cudaMemsetAsync(op->invd.p, 0, (size_t)n * 8, st));
    hbk::jacobi_diag_kernel<<<num_sms() * 8, 256, 0, st>>>(op->G.as<double>(), op->idx.as<int32_t>(),
                                                           op->mass_mode == 1 ? op->B.as<double>() : nullptr, E, op->N,
                                                           op->lam, op->invd.as<double>());
    CU_TRY(cudaGetLastError());
    hbk::invert_kernel<<<num_sms() * 8, 256, 0, st>>>(op->invd.as<double>(), n, op->mass_mode == 0 ? op->lam : 0.0);
    CU_TRY(cudaGetLastError());
    op->launches += 2;
    CU_TRY(cudaStreamSynchronize(st));
  }
  if ((enable != 0) != op->jacobi) {  // captured graphs bake the kernel arguments in
    for (auto& kv : op->graphs) cudaGraphExecDestroy(kv.second.exec);
    op->graphs.clear();
    for (auto& kv : op->tol_graphs) cudaGraphExecDestroy(kv.second.exec);
    op->tol_graphs.clear();
  }
  op->jacobi = enable != 0;
  return HB_OK;
}

extern "C" int hb_op_jacobi_diagonal(hb_op* op, double* diag_dev, void* stream) {
  if (!op || (op->sz.n_owned > 0 && !diag_dev)) { set_error("hb_op_jacobi_diagonal: null pointer"); return HB_ERR_ARG; }
  if (!op->invd.p) { set_error("hb_op_jacobi_diagonal: call hb_op_set_jacobi(op, 1) first"); return HB_ERR_STATE; }
  const int64_t n = op->sz.n_owned;
  CU_TRY(cudaMemcpyAsync(diag_dev, op->invd.p, (size_t)n * 8, cudaMemcpyDeviceToDevice, (cudaStream_t)stream));
  hbk::invert_kernel<<<num_sms() * 8, 256, 0, (cudaStream_t)stream>>>(diag_dev, n, 0.0);
  CU_TRY(cudaGetLastError());
  return HB_OK;
}

extern "C" int hb_op_set_tolerance_loop(hb_op* op, int device) {
  if (!op || (device != 0 && device != 1)) { set_error("hb_op_set_tolerance_loop: bad argument"); return HB_ERR_ARG; }
  op->tol_device_loop = device == 1;
  return HB_OK;
}

extern "C" int hb_op_set_timing_mode(hb_op* op, int mode) {
  if (!op || (mode != 0 && mode != 1)) { set_error("hb_op_set_timing_mode: bad argument"); return HB_ERR_ARG; }
  op->timing_vec_only = mode == 1;
  return HB_OK;
}

extern "C" int hb_op_launch_shape(const hb_op* op, int32_t out[4]) {
  if (!op || !out) { set_error("hb_op_launch_shape: null pointer"); return HB_ERR_ARG; }
  out[0] = op->ax_plain.grid_max;
  out[1] = op->ax_plain.block;
  out[2] = op->ax_plain.epb;
  out[3] = (int32_t)op->ax_plain.smem;
  return HB_OK;
}

extern "C" int hb_op_set_profiling(hb_op* op, int enable) {
  if (!op || enable < 0) { set_error("hb_op_set_profiling: bad argument"); return HB_ERR_ARG; }
  const bool on = enable != 0;
  if (on != op->profiling || (on && enable != op->prof_stride)) {
    // captured graphs bake the event pattern in: drop them when it changes
    for (auto& kv : op->graphs) cudaGraphExecDestroy(kv.second.exec);
    op->graphs.clear();
  }
  op->profiling = on;
  op->prof_stride = on ? enable : 1;
  op->prof_seq = 0;
  op->prof_used = 0;
  op->t_xr.used = 0;
  op->t_p.used = 0;
  return HB_OK;
}

extern "C" int hb_op_kernel_time(hb_op* op, int64_t* launches, double* mean_seconds) {
  if (!op || !launches || !mean_seconds) { set_error("hb_op_kernel_time: null pointer"); return HB_ERR_ARG; }
  double tot = 0.0;
  for (size_t t = 0; t < op->prof_used; ++t) {
    float ms = 0.f;
    CU_TRY(cudaEventSynchronize(op->prof_events[t].second));
    CU_TRY(cudaEventElapsedTime(&ms, op->prof_events[t].first, op->prof_events[t].second));
    tot += ms * 1e-3;
  }
  *launches = (int64_t)op->prof_used;
  *mean_seconds = op->prof_used ? tot / op->prof_used : 0.0;
  return HB_OK;
}

extern "C" int hb_op_phase_times(hb_op* op, double* mean_seconds3) {
  if (!op || !mean_seconds3) { set_error("hb_op_phase_times: null pointer"); return HB_ERR_ARG; }
  int64_t n = 0;
  HB_TRY(hb_op_kernel_time(op, &n, &mean_seconds3[0]));
  hb_op::Timer* tms[2] = {&op->t_xr, &op->t_p};
  for (int k = 0; k < 2; ++k) {
    double tot = 0.0;
    for (size_t t = 0; t < tms[k]->used; ++t) {
      float ms = 0.f;
      CU_TRY(cudaEventSynchronize(tms[k]->ev[t].second));
      CU_TRY(cudaEventElapsedTime(&ms, tms[k]->ev[t].first, tms[k]->ev[t].second));
      tot += ms * 1e-3;
    }
    mean_seconds3[1 + k] = tms[k]->used ? tot / tms[k]->used : 0.0;
  }
  return HB_OK;
}

extern "C" int hb_op_launch_count(hb_op* op, int64_t* launches) {
  if (!op || !launches) { set_error("hb_op_launch_count: null pointer"); return HB_ERR_ARG; }
  *launches = op->launches;
  return HB_OK;
}

extern "C" int hb_op_sizes(const hb_op* op, hb_sizes* out) {
  if (!op || !out) { set_error("hb_op_sizes: null pointer"); return HB_ERR_ARG; }
  *out = op->sz;
  return HB_OK;
}

extern "C" int hb_op_destroy(hb_op* op) {
  if (op) cudaDeviceSynchronize();
  delete op;
  return HB_OK;
}

// ------------------------------------------------------------------ loopback groups
struct hb_group {
  std::vector<hb_op*> ops;
  std::vector<cudaStream_t> st, cs;  // per virtual rank: compute and communication streams
  std::vector<cudaEvent_t> done;     // per virtual rank: end of its apply
  cudaEvent_t start = nullptr;
  DevBuf sums;                       // pointer table of the allreduce stand-in
  ~hb_group() {
    for (cudaStream_t x : st) cudaStreamDestroy(x);
    for (cudaStream_t x : cs) cudaStreamDestroy(x);
    for (cudaEvent_t e : done) cudaEventDestroy(e);
    if (start) cudaEventDestroy(start);
  }
};

extern "C" int hb_group_create(hb_op* const* ops, int P, hb_group** out) {
  if (!ops || !out || P < 1) { set_error("hb_group_create: bad argument"); return HB_ERR_ARG; }
  *out = nullptr;
  auto* g = new (std::nothrow) hb_group();
  if (!g) { set_error("hb_group_create: out of memory"); return HB_ERR_OOM; }
  for (int r = 0; r < P; ++r) {
    if (!ops[r] || ops[r]->sz.P != P || ops[r]->sz.rank != r || ops[r]->comm) {
      set_error("hb_group_create: ops must be the P comm-less ops of one partition, in rank order");
      delete g; return HB_ERR_STATE;
    }
    g->ops.push_back(ops[r]);
  }
  // plan consistency: what r sends to q is what q expects from r
  for (int r = 0; r < P; ++r) {
    hb_op* a = g->ops[r];
    for (size_t q = 0; q < a->nbr.size(); ++q) {
      hb_op* b = g->ops[a->nbr[q]];
      auto itq = std::find(b->nbr.begin(), b->nbr.end(), r);
      if (itq == b->nbr.end()) { set_error("hb_group_create: asymmetric neighbour sets"); delete g; return HB_ERR_SETUP; }
      const size_t back = (size_t)(itq - b->nbr.begin());
      if (a->scnt[q] != b->rcnt[back] || a->rcnt[q] != b->scnt[back]) {
        set_error("hb_group_create: send/recv plan sizes disagree"); delete g; return HB_ERR_SETUP;
      }
    }
  }
  int lo = 0, hi = 0;
  cudaDeviceGetStreamPriorityRange(&lo, &hi);
  g->st.resize(P); g->cs.resize(P); g->done.resize(P);
  for (int r = 0; r < P; ++r) {
    if (cudaStreamCreateWithFlags(&g->st[r], cudaStreamNonBlocking) != cudaSuccess ||
        cudaStreamCreateWithPriority(&g->cs[r], cudaStreamNonBlocking, hi) != cudaSuccess ||
        cudaEventCreateWithFlags(&g->done[r], cudaEventDisableTiming) != cudaSuccess) {
      set_error("hb_group_create: stream/event creation failed"); delete g; return HB_ERR_CUDA;
    }
    g->ops[r]->grouped = true;
  }
  if (cudaEventCreateWithFlags(&g->start, cudaEventDisableTiming) != cudaSuccess) {
    set_error("hb_group_create: event creation failed"); delete g; return HB_ERR_CUDA;
  }
  int st = g->sums.alloc(8 * P);
  if (st) { delete g; return st; }
  *out = g;
  return HB_OK;
}

namespace {
// Loopback transport: rank r pulls each message addressed to it from the sender's buffer on
// r's communication stream, after the sender's data-ready event (ev_pack for the halo
// exchange, ev_haloel for the assembly exchange) -- the same message lists NCCL gets.
int loopback_exchange(hb_group* g, int r, int kind, cudaStream_t cs) {
  hb_op* a = g->ops[r];
  std::vector<Msg> snd, rcv, psnd, prcv;
  if (kind == 0) halo_msgs(a, snd, rcv); else assembly_msgs(a, snd, rcv);
  for (const Msg& m : rcv) {
    hb_op* b = g->ops[m.peer];
    if (kind == 0) halo_msgs(b, psnd, prcv); else assembly_msgs(b, psnd, prcv);
    const Msg* match = nullptr;
    for (const Msg& ps : psnd) if (ps.peer == r) match = &ps;
    if (!match || match->count != m.count) { set_error("loopback_exchange: unmatched message"); return HB_ERR_SETUP; }
    CU_TRY(cudaStreamWaitEvent(cs, kind == 0 ? b->ev_pack : b->ev_haloel, 0));
    CU_TRY(cudaMemcpyAsync(m.buf, match->buf, (size_t)m.count * 8, cudaMemcpyDeviceToDevice, cs));
  }
  return HB_OK;
}

// The split apply of all virtual ranks, each on its own compute + communication stream with
// the NCCL path's events: packs first (so every data-ready event exists before anyone waits
// on it), then every rank's halo phase, then every rank's assembly phase.
int group_apply_internal(hb_group* g, const double* const* x, double* const* y, bool init_y, cudaStream_t st,
                         bool energy = false) {
  const int P = (int)g->ops.size();
  CU_TRY(cudaEventRecord(g->start, st));
  for (int r = 0; r < P; ++r) {
    CU_TRY(cudaStreamWaitEvent(g->st[r], g->start, 0));
    HB_TRY(stage_init(g->ops[r], x[r], y[r], init_y, g->st[r]));
    CU_TRY(cudaEventRecord(g->ops[r]->ev_pack, g->st[r]));
  }
  for (int r = 0; r < P; ++r) {
    auto ex = [g, r](int kind, cudaStream_t c) { return loopback_exchange(g, r, kind, c); };
    HB_TRY(rank_phase_halo(g->ops[r], x[r], y[r], g->st[r], g->cs[r], energy, last_launch(g->ops[r]), ex));
  }
  for (int r = 0; r < P; ++r) {
    auto ex = [g, r](int kind, cudaStream_t c) { return loopback_exchange(g, r, kind, c); };
    HB_TRY(rank_phase_assembly(g->ops[r], x[r], y[r], g->st[r], g->cs[r], energy, last_launch(g->ops[r]), ex));
    CU_TRY(cudaEventRecord(g->done[r], g->st[r]));
  }
  for (int r = 0; r < P; ++r) CU_TRY(cudaStreamWaitEvent(st, g->done[r], 0));
  return HB_OK;
}

__global__ void group_sum_kernel(double* const* parts, int P, double* const* dsts) {
  // every rank receives the rank-ordered sum of the P local values (allreduce stand-in)
  double s = 0.0;
  for (int r = 0; r < P; ++r) s += *parts[r];
  for (int r = 0; r < P; ++r) *dsts[r] = s;
}

int group_allreduce(hb_group* g, size_t field_offset, cudaStream_t st) {
  const int P = (int)g->ops.size();
  std::vector<double*> ptrs(P);
  for (int r = 0; r < P; ++r) ptrs[r] = reinterpret_cast<double*>(g->ops[r]->scal.as<char>() + field_offset);
  // stage the pointer table in the group's scratch (P doubles reinterpreted as pointers)
  CU_TRY(cudaMemcpyAsync(g->sums.p, ptrs.data(), P * sizeof(double*), cudaMemcpyHostToDevice, st));
  double* const* table = g->sums.as<double*>();
  group_sum_kernel<<<1, 1, 0, st>>>(table, P, table);
  CU_TRY(cudaGetLastError());
  return HB_OK;
}
}  // namespace

extern "C" int hb_group_apply(hb_group* g, const double* const* x, double* const* y, void* stream) {
  if (!g || !x || !y) { set_error("hb_group_apply: null pointer"); return HB_ERR_ARG; }
  return group_apply_internal(g, x, y, true, (cudaStream_t)stream);
}

extern "C" int hb_group_cg_solve(hb_group* g, const double* const* b, double* const* x, int32_t max_iters, double eps,
                                 double* rr_hist_host, hb_cg_result* res, void* stream) {
  if (!g || !b || !x || max_iters < 0) { set_error("hb_group_cg_solve: bad argument"); return HB_ERR_ARG; }
  cudaStream_t st = (cudaStream_t)stream;
  const int P = (int)g->ops.size();
  for (int r = 0; r < P; ++r) HB_TRY(ensure_hist(g->ops[r], max_iters));
  const size_t off_pAp = offsetof(hbk::CgScalars, pAp), off_rrn = offsetof(hbk::CgScalars, rr_new),
               off_rrl = offsetof(hbk::CgScalars, rr_loc);
  for (int r = 0; r < P; ++r) HB_TRY(cg_init(g->ops[r], b[r], x[r], st));
  HB_TRY(group_allreduce(g, off_rrn, st));
  hb_op* o0 = g->ops[0];
  hbk::CgScalars* hs = reinterpret_cast<hbk::CgScalars*>(o0->host_scal);
  auto read0 = [&]() -> int {
    CU_TRY(cudaMemcpyAsync(o0->host_scal, o0->scal.p, sizeof(hbk::CgScalars), cudaMemcpyDeviceToHost, st));
    CU_TRY(cudaStreamSynchronize(st));
    return HB_OK;
  };
  HB_TRY(read0());
  double rr = hs->rr_new;
  int32_t j = 0;
  std::vector<const double*> pv(P);
  std::vector<double*> av(P);
  for (int r = 0; r < P; ++r) { pv[r] = g->ops[r]->p.as<double>(); av[r] = g->ops[r]->Ap.as<double>(); }
  while (j < max_iters && (eps < 0 || rr > eps)) {
    HB_TRY(group_apply_internal(g, pv.data(), av.data(), false, st, true));
    HB_TRY(group_allreduce(g, off_pAp, st));
    for (int r = 0; r < P; ++r) {  // same split as the NCCL path: r update + r.r, then x AXPY
      hb_op* a = g->ops[r];
      const int64_t n = a->sz.n_owned;
      hbk::cg_update_r<<<vec_grid(std::max<int64_t>(n, 1)), hbk::VEC_BLOCK, 0, st>>>(
          a->r.as<double>(), a->Ap.as<double>(), n, a->partials.as<double>(), a->scal.as<hbk::CgScalars>());
    }
    HB_TRY(group_allreduce(g, off_rrl, st));
    for (int r = 0; r < P; ++r) {
      hb_op* a = g->ops[r];
      const int64_t n = a->sz.n_owned;
      hbk::cg_update_x<<<vec_grid(std::max<int64_t>(n, 1)), hbk::VEC_BLOCK, 0, st>>>(
          x[r], a->p.as<double>(), n, a->scal.as<hbk::CgScalars>());
    }
    if (eps >= 0) {
      HB_TRY(read0());
      if (!(hs->pAp > 0.0) || !std::isfinite(hs->pAp) || !std::isfinite(hs->rr_loc)) {
        set_error("hb_group_cg_solve: breakdown"); return HB_ERR_BREAKDOWN;
      }
      rr = hs->rr_loc;
    }
    for (int r = 0; r < P; ++r) HB_TRY(cg_vec_part2(g->ops[r], st));
    ++j;
  }
  return finish_result(o0, j, rr_hist_host, res, st);
}

extern "C" int hb_group_destroy(hb_group* g) {
  if (g) for (hb_op* o : g->ops) o->grouped = false;
  delete g;
  return HB_OK;
}

// ------------------------------------------------------------------ 8:1 streaming calibration
extern "C" int hb_stream_bench(int64_t n_out, int reps, double* bytes_per_s) {
  if (n_out <= 0 || reps <= 0 || !bytes_per_s) { set_error("hb_stream_bench: bad argument"); return HB_ERR_ARG; }
  DevBuf in, out;
  HB_TRY(in.alloc((size_t)n_out * 8 * 8));
  HB_TRY(out.alloc((size_t)n_out * 8));
  CU_TRY(cudaMemset(in.p, 0, (size_t)n_out * 64));
  cudaEvent_t e0, e1;
  CU_TRY(cudaEventCreate(&e0));
  CU_TRY(cudaEventCreate(&e1));
  const int grid = num_sms() * 8;
  for (int w = 0; w < 3; ++w) hbk::stream8to1<<<grid, hbk::VEC_BLOCK>>>(in.as<double>(), out.as<double>(), n_out);
  CU_TRY(cudaEventRecord(e0));
  for (int t = 0; t < reps; ++t) hbk::stream8to1<<<grid, hbk::VEC_BLOCK>>>(in.as<double>(), out.as<double>(), n_out);
  CU_TRY(cudaEventRecord(e1));
  CU_TRY(cudaEventSynchronize(e1));
  float ms = 0;
  CU_TRY(cudaEventElapsedTime(&ms, e0, e1));
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  *bytes_per_s = 72.0 * (double)n_out * reps / (ms * 1e-3);
  return HB_OK;
}
