/*
 * hipbone_b200.h -- C ABI of the B200-native hipBone hot path (arXiv 2202.12477).
 *
 * The library applies the assembled spectral-element screened-Poisson operator
 *     A = Z^T (S_L + lambda M_L) Z,   S_L^e = bold-D^T G^e bold-D
 * matrix-free on a structured box of E hexahedra of degree N, and runs the
 * preconditioner-free conjugate-gradient iteration of Algorithm 1 that NekBone
 * times.  Citations P:<line> refer to the paper text; readings c<k>
 * refer to SURVEY.md §8(c) and are restated in DESIGN.md.
 *
 * Conventions (binding for every call):
 *   - All status-returning calls return HB_OK (0) or a negative HB_ERR_* code; no C++
 *     exception crosses the ABI.  hb_last_error() returns a thread-local message for the
 *     last failing call on the calling thread.
 *   - Floating point is IEEE fp64 throughout; indices at the ABI are int64 (global ids)
 *     or int32 (local indices).
 *   - Numbering (c7): element e = ex + nx (ey + ny ez); local node n = i + (N+1)(j + (N+1)k);
 *     global id of grid point (X,Y,Z) = X + (nx N + 1)(Y + (ny N + 1) Z), X = ex N + i.
 *   - "host" pointers are ordinary CPU memory; "dev" pointers are CUDA device memory
 *     (e.g. torch.cuda tensors, float64, contiguous) on the current device.
 *   - Pointer ownership: the caller owns every pointer it passes; the library owns the
 *     opaque handles (hb_mesh, hb_op, hb_comm, hb_group) and all their internal buffers,
 *     released by the matching *_destroy call.
 *   - Streams: `stream` is a cudaStream_t passed as void* (NULL = legacy default stream).
 *     Device calls are asynchronous on it unless stated otherwise.
 *   - Distributed vectors: rank r stores x[g] for g in owned(r), ascending gid
 *     ("assembled storage").  With P = 1 owned = 0..N_G-1.
 */
#ifndef HIPBONE_B200_H
#define HIPBONE_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define HB_ABI_VERSION 1

enum {
  HB_OK = 0,
  HB_ERR_ARG = -1,       /* bad argument: N outside [1,15], rank outside [0,P), null pointer, size mismatch */
  HB_ERR_CONFIG = -2,    /* no admissible rank grid (px<=nx, py<=ny, pz<=nz), c8 */
  HB_ERR_GEOMETRY = -3,  /* element extent <= 0 */
  HB_ERR_SETUP = -4,     /* inconsistent sharing / exchange plans */
  HB_ERR_STATE = -5,     /* call-order violation (e.g. op on a destroyed mesh, comm missing for P>1) */
  HB_ERR_BREAKDOWN = -6, /* CG breakdown in tolerance mode: p.Ap <= 0 or non-finite */
  HB_ERR_CUDA = -7,      /* CUDA runtime error (message carries cudaGetErrorString) */
  HB_ERR_NCCL = -8,      /* NCCL error */
  HB_ERR_OOM = -9        /* host or device allocation failed */
};

/* Box of nx*ny*nz hexahedra of degree N.  ext = element extent per axis (c4,
 * default {2,2,2}: J = 1, identity metric).  mass_mode selects M_L (c3):
 *   0 = lambda W, W = inverse degree weights, Z^T W Z = I (the paper's choice);
 *   1 = lambda B, B = w_i w_j w_k J (GLL lumped mass).                                   */
typedef struct {
  int32_t nx, ny, nz, N;
  double ext[3];
  int32_t mass_mode;
} hb_box;

typedef struct {
  int64_t E_global, E_local;   /* elements in the box / on this rank                      */
  int64_t N_L;                 /* E_local (N+1)^3 local slots                              */
  int64_t N_G;                 /* global DOFs (nx N+1)(ny N+1)(nz N+1)                     */
  int64_t n_owned, n_halo;     /* owned DOFs; non-owned DOFs referenced by local elements  */
  int64_t n_intA, n_halo_elems, n_intB; /* element classes, local order [A | halo | B]     */
  int32_t n_neighbors, rank, P, grid[3];
} hb_sizes;

typedef struct {
  int32_t iterations;          /* CG iterations performed (j of Alg. 1)                  */
  double rr0, rr_final;        /* r_0.r_0 and r_j.r_j                                     */
} hb_cg_result;

typedef struct hb_mesh hb_mesh;
typedef struct hb_comm hb_comm;
typedef struct hb_op hb_op;
typedef struct hb_group hb_group;

/* ---------------------------------------------------------------- general */
const char* hb_last_error(void);
int hb_version(void); /* returns HB_ABI_VERSION */

/* GLL nodes (ascending), weights and derivative matrix D[i*(N+1)+j] = l_j'(x_i)
 * (P:48).  Host arrays of N+1, N+1 and (N+1)^2 doubles.  HB_ERR_ARG if N<1 or N>15. */
int hb_gll(int N, double* nodes, double* weights, double* D);

/* Rank grid for P ranks (c8): minimises total cut area (px-1)ny nz + (py-1)nx nz +
 * (pz-1)nx ny subject to px<=nx, py<=ny, pz<=nz; ties prefer px>=py>=pz, then the
 * lexicographically largest.  HB_ERR_CONFIG if none exists. */
int hb_rank_grid(int P, int nx, int ny, int nz, int32_t grid_out[3]);

/* ---------------------------------------------------------------- mesh (host only, deterministic)
 * Partition (c8): remainder element layers go to the lowest ranks per axis; rank
 * r = rx + px (ry + py rz).  Ownership of shared DOFs (c9): owner(g) =
 * sorted_sharers[splitmix64(splitmix64(seed) ^ g) mod k].  Halo element: has
 * >= 1 node shared with another rank.  Local element order: [interior A | halo |
 * interior B], A = first ceil(I/2) interior elements ascending (c10).
 * Extended local vector: [owned ascending | halo grouped by owner rank, gid ascending] (c11).
 * grid = NULL picks hb_rank_grid().  No CUDA call is made. */
int hb_mesh_create(const hb_box* box, int P, int rank, const int32_t* grid, uint64_t seed,
                   hb_mesh** out);
int hb_mesh_sizes(const hb_mesh* m, hb_sizes* out);
/* global element ids in local order, [E_local] */
int hb_mesh_elements(const hb_mesh* m, int64_t* elem_ids);
/* global ids per slot, [E_local][(N+1)^3] */
int hb_mesh_l2g(const hb_mesh* m, int64_t* gid);
/* local index of every slot into the extended vector [owned | halo], [E_local][(N+1)^3] */
int hb_mesh_local_index(const hb_mesh* m, int32_t* idx);
/* owned gids ascending [n_owned]; halo gids in extended-vector order [n_halo] */
int hb_mesh_owned(const hb_mesh* m, int64_t* owned);
int hb_mesh_halo(const hb_mesh* m, int64_t* halo);
/* neighbour ranks ascending [n_neighbors] with the number of DOFs sent to / received from each */
int hb_mesh_neighbors(const hb_mesh* m, int32_t* ranks, int64_t* send_counts, int64_t* recv_counts);
/* gids this rank sends to neighbour number q (owned gids referenced by that rank, ascending) */
int hb_mesh_send_list(const hb_mesh* m, int q, int64_t* gids);
/* geometric factors, host [E_local][(N+1)^3][6] packed per node rr,rs,rt,ss,st,tt */
int hb_mesh_geometry(const hb_mesh* m, double* G);
/* override the geometric factors (test hook for random SPD factors, c6); same layout */
int hb_mesh_set_geometry(hb_mesh* m, const double* G);
/* mass per slot [E_local][(N+1)^3]: W (mode 0) or B (mode 1) */
int hb_mesh_mass(const hb_mesh* m, double* M);
/* override the mode-1 mass B (test hook); HB_ERR_STATE in mode 0 (W is topological) */
int hb_mesh_set_mass(hb_mesh* m, const double* M);
int hb_mesh_destroy(hb_mesh* m);

/* ---------------------------------------------------------------- communicator (NCCL, P>1)
 * Rank 0 calls hb_comm_unique_id and broadcasts the 128 bytes (e.g. torch.distributed);
 * every rank then calls hb_comm_create with its rank.  One GPU per rank (current device). */
int hb_comm_unique_id(uint8_t id[128]);
int hb_comm_create(int P, int rank, const uint8_t id[128], hb_comm** out);
int hb_comm_destroy(hb_comm* c);
/* Peer-memory transport (the direct-NVLink alternative to NCCL for the
 * two exchanges of P:201-203 and the CG allreduces of P:213-217): no NCCL communicator; every
 * op built on it must be connected with hb_op_ipc_connect before use.  Ranks on one node
 * (any GPUs, or several ranks on one GPU).  Data moves with peer copies into the receiver's
 * buffers (CUDA IPC mappings; NVLink copy engines across GPUs); ordering uses 32-bit sequence
 * flags in the receiver's mailbox (stream memory operations), never a host synchronisation.
 * Fixed-mode CG runs as a stream-ordered loop (no graph: the flags carry per-call sequence
 * numbers).  HB_ERR_ARG on bad (P, rank). */
int hb_comm_create_ipc(int P, int rank, hb_comm** out);

/* ---------------------------------------------------------------- operator
 * hb_op_create uploads the local index, geometric factors (and B in mode 1) and exchange
 * plans to the current device and allocates the workspace; synchronous.  comm must be
 * non-NULL iff P > 1 (unless the op is part of a loopback group).  lambda is the screening
 * coefficient of eq:poisson (c2: 1 in every benchmark config). */
int hb_op_create(const hb_mesh* m, hb_comm* comm, double lambda, void* stream, hb_op** out);
/* y_dev = A x_dev on owned DOFs ([n_owned] each, distinct device buffers).  Fused
 * gather / S_L + lambda M_L / scatter-add kernel (P:154 extended by the Z^T fusion).  Asynchronous. */
int hb_op_apply(hb_op* op, const double* x_dev, double* y_dev, void* stream);
/* IPC transport bootstrap (op on an hb_comm_create_ipc communicator).  hb_op_ipc_blob_size
 * gives the byte size B of this op's export record (same on every rank: a function of P);
 * hb_op_ipc_export writes it (CUDA IPC handles of the mailbox, the halo receive buffer and
 * the assembly receive buffer, plus the neighbour list, counts and offsets).  The caller
 * all-gathers the P records (rank order, P*B bytes) and passes them to hb_op_ipc_connect,
 * which maps every peer's mailbox and the buffers this rank writes into, and checks that the
 * plans agree (HB_ERR_STATE otherwise).  Collective: every rank calls it once. */
int hb_op_ipc_blob_size(const hb_op* op, int64_t* bytes);
int hb_op_ipc_export(const hb_op* op, uint8_t* blob);
int hb_op_ipc_connect(hb_op* op, const uint8_t* blobs);
/* IPC direct mode for CG (default on): the halo-element kernel reads the owners' p and
 * scatter-adds (fp64 RED) into the owners' Ap through per-halo-node peer pointers, so the
 * operator of a CG iteration needs no exchange, pack or unpack -- the collective is fused into
 * the compute kernel.  Ordering: per iteration each owner raises RDY after writing p and
 * Ap = lambda p; each sharer waits RDY before its halo elements and raises DONE after them;
 * the owner waits DONE before reading Ap.  enable = 0 selects the exchange path (as
 * hb_op_apply always uses).  Collective: all ranks must use the same setting. */
int hb_op_set_ipc_direct(hb_op* op, int enable);
/* b_dev[l] = forcing(owned_gid[l], seed) (c12), [n_owned].  Asynchronous. */
int hb_forcing(hb_op* op, uint64_t seed, double* b_dev, void* stream);
/* global a.b over owned DOFs (allreduced for P>1); synchronises the stream. */
int hb_dot(hb_op* op, const double* a_dev, const double* b_dev, double* out_host, void* stream);
/* CG (Alg. 1) from x_0 = 0 (c13).  eps < 0: fixed mode, exactly max_iters
 * iterations, captured in a CUDA graph; eps >= 0: tolerance mode, stop when
 * r.r <= eps (absolute, c14) or j == max_iters; HB_ERR_BREAKDOWN if p.Ap <= 0 or
 * non-finite.  With P = 1 tolerance mode is also one CUDA graph: a WHILE conditional node
 * whose loop test (r.r > eps, j < max_iters, no breakdown) runs on the device, so the host
 * synchronises only at the end (hb_op_set_tolerance_loop(op, 0) selects a host-driven loop).  rr_hist_host (nullable) receives r_j.r_j for j = 0..iterations
 * ([max_iters+1]).  x_dev receives the solution [n_owned].  Synchronises the stream at the end. */
int hb_cg_solve(hb_op* op, const double* b_dev, double* x_dev, int32_t max_iters, double eps,
                double* rr_hist_host, hb_cg_result* res, void* stream);
/* NekBone's scattered storage, for comparison with the
 * assembled storage above: CG on local vectors x_L = Z x of length N_L with the operator
 * (Z Z^T S_L + lambda I) x_L (element kernel on x_L, combined gather-scatter through a CSR
 * in ascending (e, n) order) and inner products weighted by the inverse counting vector W
 * (P:121).  Same arguments and modes as hb_cg_solve (b, x assembled [n_owned]); P = 1 and
 * mass mode 0 only (HB_ERR_STATE otherwise).  Synchronises the stream at the end. */
int hb_cg_solve_scattered(hb_op* op, const double* b_dev, double* x_dev, int32_t max_iters, double eps,
                          double* rr_hist_host, hb_cg_result* res, void* stream);
/* Same solve with HOST buffers: copies b (pinned or pageable) to the device, solves, copies
 * x back; copies are inside the call (end-to-end path). */
int hb_cg_solve_host(hb_op* op, const double* b_host, double* x_host, int32_t max_iters, double eps,
                     double* rr_hist_host, hb_cg_result* res, void* stream);
/* Assembly variant: 0 (default) = Z^T fused into the operator as fp64 scatter-add (atomic
 * accumulation order, results reproducible to rounding); 1 = the paper's split form (P:154,
 * P:219): the operator writes y_L per slot and a CSR gather kernel sums every DOF's slots in
 * ascending (e, n) order -- bitwise reproducible, +20 N_L bytes per apply.  Variant 1: P = 1
 * only (HB_ERR_STATE otherwise); HB_ERR_ARG for any other value.  Synchronous (builds the CSR
 * on first use). */
int hb_op_set_variant(hb_op* op, int variant, void* stream);
/* Jacobi-preconditioned CG (NekBone's diagonal preconditioner, P:140 --
 * hipBone itself uses none).  enable = 1 computes M = diag(A) on the device once
 * (sum over slots of (S_L^e)_nn, + lambda) and makes hb_cg_solve run PCG: alpha = r.z / p.Ap,
 * beta = r'.z' / r.z, p = z + beta p with z = M^-1 r; the stopping test stays r.r <= eps and
 * the history stays r.r.  P = 1 only (HB_ERR_STATE otherwise).  Synchronous.
 * hb_op_jacobi_diagonal writes diag(A) [n_owned] to a device buffer (test hook). */
int hb_op_set_jacobi(hb_op* op, int enable, void* stream);
int hb_op_jacobi_diagonal(hb_op* op, double* diag_dev, void* stream);
/* Tolerance-mode loop of hb_cg_solve (P = 1): device = 1 (default) runs the loop test on the
 * device inside one CUDA graph (WHILE conditional node); device = 0 runs a host-driven loop that
 * reads r.r back every iteration (the reference behaviour for tests).  HB_ERR_ARG otherwise. */
int hb_op_set_tolerance_loop(hb_op* op, int device);
/* Measurement hook for splitting a fixed-mode CG step into its kernels without instrumenting
 * it: mode = 1 makes subsequent fixed-mode hb_cg_solve calls run the same graph WITHOUT the
 * operator launches (vector kernels only; x and the history are meaningless), so that
 * (t(mode 0) - t(mode 1)) / iterations is the operator's in-situ share of an iteration
 * (an upper bound: the vector kernels alone find their vectors in L2).  mode = 0 restores
 * the solver.  HB_ERR_ARG otherwise. */
int hb_op_set_timing_mode(hb_op* op, int mode);
/* Launch shape of the operator kernel used by hb_op_apply / hb_cg_solve on the rank's
 * interior elements: out[0] = resident grid (CTAs the kernel launches at most; it loops over
 * elements beyond that), out[1] = threads per CTA, out[2] = elements per CTA per loop trip,
 * out[3] = dynamic shared memory bytes per CTA.  Host-only query (test hook: parity cases
 * size their meshes to several grid waves). */
int hb_op_launch_shape(const hb_op* op, int32_t out[4]);
/* Profiling of the operator kernel inside hb_cg_solve / hb_op_apply: enable = k > 0 brackets
 * every k-th operator launch with CUDA events on its stream (inside captured graphs as event
 * nodes); enable = 0 turns it off.  hb_op_kernel_time returns the number of timed launches
 * of the last solve (or since enabling, outside graphs) and their mean duration in seconds. */
int hb_op_set_profiling(hb_op* op, int enable);
int hb_op_kernel_time(hb_op* op, int64_t* launches, double* mean_seconds);
/* Mean durations (seconds) of the timed CG phases of the last solve: [0] operator,
 * [1] x/r update (with the p.Ap reduction), [2] p update; 0 for a phase never timed (P > 1
 * vector phases are not timed). */
int hb_op_phase_times(hb_op* op, double* mean_seconds3);
/* Launch statistics: number of library kernels launched since creation. */
int hb_op_launch_count(hb_op* op, int64_t* launches);
int hb_op_sizes(const hb_op* op, hb_sizes* out);
int hb_op_destroy(hb_op* op);

/* ---------------------------------------------------------------- loopback group
 * P virtual ranks in one process on one GPU (test mode for the multi-rank schedule):
 * the ops are created with comm = NULL from the P meshes of one partition; exchanges
 * become device-to-device copies between the ranks' buffers, dots are summed in rank order.
 * Vector arguments are arrays of P device pointers (one owned vector per rank). */
int hb_group_create(hb_op* const* ops, int P, hb_group** out);
int hb_group_apply(hb_group* g, const double* const* x_dev, double* const* y_dev, void* stream);
int hb_group_cg_solve(hb_group* g, const double* const* b_dev, double* const* x_dev, int32_t max_iters,
                      double eps, double* rr_hist_host, hb_cg_result* res, void* stream);
int hb_group_destroy(hb_group* g);

/* ---------------------------------------------------------------- calibration
 * 8:1 streaming kernel: each thread reads 8 fp64 and writes 1; n_out outputs,
 * reps timed repetitions after 3 warm-ups; returns bytes moved (72 n_out) / mean time. */
int hb_stream_bench(int64_t n_out, int reps, double* bytes_per_s);

#ifdef __cplusplus
}
#endif
#endif /* HIPBONE_B200_H */
