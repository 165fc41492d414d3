// Host-side setup of the hipBone hot path: GLL basis, structured box mesh, element
// partition, ownership of shared DOFs, halo/interior classification and the exchange
// plans (hb_mesh_* of include/hipbone_b200.h).  Deterministic, no CUDA.
//
// P:55      regular box of E hexahedra, (N+1)^3 points per element, N_L = E (N+1)^3
// P:167     mesh partitioned evenly among the P processes (rule c8)
// P:190-192 halo node / halo element / interior element
// P:201     owner of a shared node "chosen randomly, but fairly" (rule c9)
// P:201-203 interior elements split in halves around the halo elements (rule c10)
#include <algorithm>
#include <climits>
#include <cmath>
#include <cstring>
#include <mutex>
#include <new>

#include "internal.h"

namespace {
thread_local std::string g_err;
}

namespace hb {
void set_error(const std::string& msg) { g_err = msg; }

static void legendre_pair(int N, double x, double& pN, double& pN1, double& dpN) {
  // P_N, P_{N-1} by recurrence; P_N' from (1-x^2) P_N' = N (P_{N-1} - x P_N) off the ends.
  double p0 = 1.0, p1 = x;
  if (N == 0) { pN = 1.0; pN1 = 0.0; dpN = 0.0; return; }
  for (int k = 1; k < N; ++k) {
    double p2 = ((2.0 * k + 1.0) * x * p1 - k * p0) / (k + 1.0);
    p0 = p1; p1 = p2;
  }
  pN = p1; pN1 = p0;
  dpN = N * (pN1 - x * pN) / (1.0 - x * x);
}

void gll_basis(int N, std::vector<double>& x, std::vector<double>& w, std::vector<double>& D) {
  const int NP = N + 1;
  x.assign(NP, 0.0); w.assign(NP, 0.0); D.assign(NP * NP, 0.0);
  x[0] = -1.0; x[N] = 1.0;
  // interior nodes: roots of P_N'.  Newton on f = P_N' with f' = (2x P_N' - N(N+1) P_N)/(1-x^2).
  for (int i = 1; i < N; ++i) {
    double xi = -std::cos(M_PI * i / N);
    for (int it = 0; it < 100; ++it) {
      double pN, pN1, dpN;
      legendre_pair(N, xi, pN, pN1, dpN);
      double d2 = (2.0 * xi * dpN - N * (N + 1.0) * pN) / (1.0 - xi * xi);
      double dx = dpN / d2;
      xi -= dx;
      if (std::fabs(dx) < 1e-16) break;
    }
    x[i] = xi;
  }
  for (int i = 0; i < NP / 2; ++i) {  // exact symmetry
    double a = 0.5 * (x[N - i] - x[i]);
    x[i] = -a; x[N - i] = a;
  }
  if (N % 2 == 0) x[N / 2] = 0.0;
  std::vector<double> PN(NP);
  for (int i = 0; i < NP; ++i) {
    double pN, pN1, dpN;
    if (i == 0 || i == N) {  // P_N(+-1) = (+-1)^N
      pN = (i == 0 && (N % 2)) ? -1.0 : 1.0;
    } else {
      legendre_pair(N, x[i], pN, pN1, dpN);
    }
    PN[i] = pN;
    w[i] = 2.0 / (N * (N + 1.0) * pN * pN);
  }
  for (int i = 0; i < NP; ++i)
    for (int j = 0; j < NP; ++j) {
      double v;
      if (i != j) v = PN[i] / (PN[j] * (x[i] - x[j]));
      else if (i == 0) v = -N * (N + 1.0) / 4.0;
      else if (i == N) v = N * (N + 1.0) / 4.0;
      else v = 0.0;
      D[i * NP + j] = v;
    }
}
}  // namespace hb

using hb::set_error;

extern "C" const char* hb_last_error(void) { return g_err.c_str(); }
extern "C" int hb_version(void) { return HB_ABI_VERSION; }

extern "C" int hb_gll(int N, double* nodes, double* weights, double* D) {
  if (N < 1 || N > 15) { set_error("hb_gll: N must be in [1,15]"); return HB_ERR_ARG; }
  if (!nodes || !weights || !D) { set_error("hb_gll: null pointer"); return HB_ERR_ARG; }
  std::vector<double> x, w, d;
  hb::gll_basis(N, x, w, d);
  std::memcpy(nodes, x.data(), x.size() * 8);
  std::memcpy(weights, w.data(), w.size() * 8);
  std::memcpy(D, d.data(), d.size() * 8);
  return HB_OK;
}

extern "C" int hb_rank_grid(int P, int nx, int ny, int nz, int32_t grid_out[3]) {
  if (P < 1 || nx < 1 || ny < 1 || nz < 1 || !grid_out) { set_error("hb_rank_grid: bad argument"); return HB_ERR_ARG; }
  bool found = false;
  int64_t best_area = 0; int best_ord = 0, bx = 0, by = 0, bz = 0;
  for (int px = 1; px <= P; ++px) {
    if (P % px) continue;
    for (int py = 1; py <= P / px; ++py) {
      if ((P / px) % py) continue;
      int pz = P / px / py;
      if (px > nx || py > ny || pz > nz) continue;
      int64_t area = (int64_t)(px - 1) * ny * nz + (int64_t)(py - 1) * nx * nz + (int64_t)(pz - 1) * nx * ny;
      int ord = (px >= py && py >= pz) ? 0 : 1;
      bool better = !found || area < best_area || (area == best_area && ord < best_ord) ||
                    (area == best_area && ord == best_ord &&
                     (px > bx || (px == bx && (py > by || (py == by && pz > bz)))));
      if (better) { found = true; best_area = area; best_ord = ord; bx = px; by = py; bz = pz; }
    }
  }
  if (!found) {
    set_error("hb_rank_grid: no factorisation of P=" + std::to_string(P) + " with px<=" + std::to_string(nx) +
              ", py<=" + std::to_string(ny) + ", pz<=" + std::to_string(nz));
    return HB_ERR_CONFIG;
  }
  grid_out[0] = bx; grid_out[1] = by; grid_out[2] = bz;
  return HB_OK;
}

namespace {
// first layer owned by rank coordinate q when n layers are split over p (remainder low)
inline int64_t layer_start(int64_t n, int p, int q) {
  int64_t base = n / p, rem = n % p;
  return q * base + std::min<int64_t>(q, rem);
}
inline int layer_rank(int64_t n, int p, int64_t layer) {
  int64_t base = n / p, rem = n % p;
  int64_t big = rem * (base + 1);
  if (layer < big) return (int)(layer / (base + 1));
  return (int)(rem + (layer - big) / base);
}
// rank coordinates (ascending, deduplicated) of the elements containing point coordinate X
inline int axis_sharers(int64_t X, int64_t n_el, int N, int p, int out[2]) {
  int64_t e_hi = X / N;
  int cnt = 0;
  if (X % N == 0 && X > 0) out[cnt++] = layer_rank(n_el, p, X / N - 1);
  if (e_hi < n_el) {
    int r = layer_rank(n_el, p, e_hi);
    if (cnt == 0 || out[0] != r) out[cnt++] = r;
  }
  return cnt;
}
}  // namespace

extern "C" int hb_mesh_create(const hb_box* box, int P, int rank, const int32_t* grid, uint64_t seed,
                              hb_mesh** out) {
  if (!box || !out) { set_error("hb_mesh_create: null pointer"); return HB_ERR_ARG; }
  *out = nullptr;
  const int N = box->N;
  if (N < 1 || N > 15) { set_error("hb_mesh_create: N must be in [1,15]"); return HB_ERR_ARG; }
  if (box->nx < 1 || box->ny < 1 || box->nz < 1) { set_error("hb_mesh_create: element counts must be >= 1"); return HB_ERR_ARG; }
  if (P < 1 || rank < 0 || rank >= P) { set_error("hb_mesh_create: rank must be in [0,P)"); return HB_ERR_ARG; }
  if (!(box->ext[0] > 0) || !(box->ext[1] > 0) || !(box->ext[2] > 0)) { set_error("hb_mesh_create: element extent must be > 0"); return HB_ERR_GEOMETRY; }
  if (box->mass_mode != 0 && box->mass_mode != 1) { set_error("hb_mesh_create: mass_mode must be 0 or 1"); return HB_ERR_ARG; }
  int32_t g[3];
  if (grid) {
    g[0] = grid[0]; g[1] = grid[1]; g[2] = grid[2];
    if (g[0] < 1 || g[1] < 1 || g[2] < 1 || (int64_t)g[0] * g[1] * g[2] != P || g[0] > box->nx || g[1] > box->ny || g[2] > box->nz) {
      set_error("hb_mesh_create: grid inconsistent with P or the box"); return HB_ERR_CONFIG;
    }
  } else {
    int st = hb_rank_grid(P, box->nx, box->ny, box->nz, g);
    if (st) return st;
  }
  hb_mesh* m = new (std::nothrow) hb_mesh();
  if (!m) { set_error("hb_mesh_create: out of memory"); return HB_ERR_OOM; }
  try {
    m->box = *box; m->P = P; m->rank = rank; m->seed = seed;
    m->grid[0] = g[0]; m->grid[1] = g[1]; m->grid[2] = g[2];
    m->NP = N + 1; m->NP3 = m->NP * m->NP * m->NP;
    const int64_t nx = box->nx, ny = box->ny, nz = box->nz;
    m->E_global = nx * ny * nz;
    const int64_t gx = nx * N + 1, gy = ny * N + 1, gz = nz * N + 1;
    m->NG = gx * gy * gz;
    hb::gll_basis(N, m->x, m->w, m->D);

    const int rx = rank % g[0], ry = (rank / g[0]) % g[1], rz = rank / (g[0] * g[1]);
    const int64_t ex0 = layer_start(nx, g[0], rx), ex1 = layer_start(nx, g[0], rx + 1);
    const int64_t ey0 = layer_start(ny, g[1], ry), ey1 = layer_start(ny, g[1], ry + 1);
    const int64_t ez0 = layer_start(nz, g[2], rz), ez1 = layer_start(nz, g[2], rz + 1);
    const int64_t lx = ex1 - ex0, ly = ey1 - ey0, lz = ez1 - ez0;
    const int64_t El = lx * ly * lz;
    // point box of this rank
    const int64_t X0 = ex0 * N, Y0 = ey0 * N, Z0 = ez0 * N;
    const int64_t bx = lx * N + 1, byy = ly * N + 1, bz = lz * N + 1;
    const int64_t npts = bx * byy * bz;
    if (npts >= INT32_MAX) { set_error("hb_mesh_create: local point count exceeds int32"); delete m; return HB_ERR_ARG; }

    // per point: owner rank and shared flag; local index
    std::vector<int32_t> local(npts);
    std::vector<uint8_t> shared(npts);
    std::vector<int32_t> owner(npts);
    const uint64_t hseed = hb::splitmix64(seed);
    std::vector<int> nbr_mark(P, 0);
    int64_t n_owned = 0;
    std::vector<std::pair<int32_t, int64_t>> halo_pts;  // (owner, gid)
    std::vector<int64_t> halo_lp;
    for (int64_t pz = 0; pz < bz; ++pz) {
      int sz[2]; int nzs = axis_sharers(Z0 + pz, nz, N, g[2], sz);
      for (int64_t py = 0; py < byy; ++py) {
        int sy[2]; int nys = axis_sharers(Y0 + py, ny, N, g[1], sy);
        for (int64_t px = 0; px < bx; ++px) {
          int sx[2]; int nxs = axis_sharers(X0 + px, nx, N, g[0], sx);
          const int64_t lp = px + bx * (py + byy * pz);
          const int64_t gid = (X0 + px) + gx * ((Y0 + py) + gy * (Z0 + pz));
          int k = nxs * nys * nzs;
          int own;
          if (k == 1) {
            own = sx[0] + g[0] * (sy[0] + g[1] * sz[0]);
            shared[lp] = 0;
          } else {
            int s[8]; int c = 0;
            for (int a = 0; a < nzs; ++a)
              for (int b = 0; b < nys; ++b)
                for (int d = 0; d < nxs; ++d) s[c++] = sx[d] + g[0] * (sy[b] + g[1] * sz[a]);
            std::sort(s, s + c);
            own = s[hb::splitmix64(hseed ^ (uint64_t)gid) % (uint64_t)c];
            shared[lp] = 1;
            for (int t = 0; t < c; ++t) if (s[t] != rank) nbr_mark[s[t]] = 1;
          }
          owner[lp] = own;
          if (own == rank) {
            local[lp] = (int32_t)n_owned++;
          } else {
            halo_pts.push_back({own, gid});
            halo_lp.push_back(lp);
          }
        }
      }
    }
    // owned gids ascending (iteration order is ascending gid)
    m->owned.resize(n_owned);
    for (int64_t pz = 0, t = 0; pz < bz; ++pz)
      for (int64_t py = 0; py < byy; ++py)
        for (int64_t px = 0; px < bx; ++px) {
          int64_t lp = px + bx * (py + byy * pz);
          if (owner[lp] == rank) m->owned[t++] = (X0 + px) + gx * ((Y0 + py) + gy * (Z0 + pz));
        }
    // halo ordered by (owner, gid)
    std::vector<int64_t> perm(halo_pts.size());
    for (size_t t = 0; t < perm.size(); ++t) perm[t] = (int64_t)t;
    std::stable_sort(perm.begin(), perm.end(), [&](int64_t a, int64_t b) { return halo_pts[a] < halo_pts[b]; });
    m->halo.resize(perm.size());
    for (size_t t = 0; t < perm.size(); ++t) {
      m->halo[t] = halo_pts[perm[t]].second;
      local[halo_lp[perm[t]]] = (int32_t)(n_owned + (int64_t)t);
    }
    if (n_owned + (int64_t)m->halo.size() >= INT32_MAX) { set_error("hb_mesh_create: extended vector exceeds int32"); delete m; return HB_ERR_ARG; }
    // neighbours and plans
    for (int q = 0; q < P; ++q) if (nbr_mark[q]) m->nbr.push_back(q);
    const size_t nn = m->nbr.size();
    std::vector<int> nbr_index(P, -1);
    for (size_t t = 0; t < nn; ++t) nbr_index[m->nbr[t]] = (int)t;
    m->recv_off.assign(nn, 0); m->recv_cnt.assign(nn, 0);
    for (size_t t = 0; t < m->halo.size(); ++t) m->recv_cnt[nbr_index[halo_pts[perm[t]].first]]++;
    for (size_t t = 1; t < nn; ++t) m->recv_off[t] = m->recv_off[t - 1] + m->recv_cnt[t - 1];
    m->send_loc.assign(nn, {}); m->send_gid.assign(nn, {});
    for (int64_t pz = 0; pz < bz; ++pz) {
      int sz[2]; int nzs = axis_sharers(Z0 + pz, nz, N, g[2], sz);
      for (int64_t py = 0; py < byy; ++py) {
        int sy[2]; int nys = axis_sharers(Y0 + py, ny, N, g[1], sy);
        for (int64_t px = 0; px < bx; ++px) {
          int64_t lp = px + bx * (py + byy * pz);
          if (!shared[lp] || owner[lp] != rank) continue;
          int sx[2]; int nxs = axis_sharers(X0 + px, nx, N, g[0], sx);
          int64_t gid = (X0 + px) + gx * ((Y0 + py) + gy * (Z0 + pz));
          int s[8]; int c = 0;
          for (int a = 0; a < nzs; ++a)
            for (int b = 0; b < nys; ++b)
              for (int d = 0; d < nxs; ++d) s[c++] = sx[d] + g[0] * (sy[b] + g[1] * sz[a]);
          std::sort(s, s + c);
          for (int t = 0; t < c; ++t) {
            if (s[t] == rank) continue;
            int qi = nbr_index[s[t]];
            m->send_loc[qi].push_back(local[lp]);
            m->send_gid[qi].push_back(gid);
          }
        }
      }
    }
    // element classification and local order [A | halo | B]
    const int NP = m->NP, NP3 = m->NP3;
    std::vector<int64_t> interior, halo_e;
    for (int64_t ez = ez0; ez < ez1; ++ez)
      for (int64_t ey = ey0; ey < ey1; ++ey)
        for (int64_t ex = ex0; ex < ex1; ++ex) {
          bool h = false;
          if (P > 1) {
            const int64_t bx0 = (ex - ex0) * N, by0 = (ey - ey0) * N, bz0 = (ez - ez0) * N;
            for (int k = 0; k < NP && !h; ++k)
              for (int j = 0; j < NP && !h; ++j)
                for (int i = 0; i < NP; ++i)
                  if (shared[(bx0 + i) + bx * ((by0 + j) + byy * (bz0 + k))]) { h = true; break; }
          }
          int64_t e = ex + nx * (ey + ny * ez);
          (h ? halo_e : interior).push_back(e);
        }
    const int64_t nI = (int64_t)interior.size();
    const int64_t nA = (nI + 1) / 2;
    m->nA = nA; m->nH = (int64_t)halo_e.size(); m->nB = nI - nA;
    m->elems.reserve(El);
    m->elems.insert(m->elems.end(), interior.begin(), interior.begin() + nA);
    m->elems.insert(m->elems.end(), halo_e.begin(), halo_e.end());
    m->elems.insert(m->elems.end(), interior.begin() + nA, interior.end());
    // local index per slot
    m->idx.resize((size_t)El * NP3);
    for (int64_t le = 0; le < El; ++le) {
      int64_t e = m->elems[le];
      int64_t ex = e % nx, ey = (e / nx) % ny, ez = e / (nx * ny);
      const int64_t bx0 = (ex - ex0) * N, by0 = (ey - ey0) * N, bz0 = (ez - ez0) * N;
      int32_t* row = &m->idx[(size_t)le * NP3];
      for (int k = 0; k < NP; ++k)
        for (int j = 0; j < NP; ++j)
          for (int i = 0; i < NP; ++i)
            row[i + NP * (j + NP * k)] = local[(bx0 + i) + bx * ((by0 + j) + byy * (bz0 + k))];
    }
  } catch (const std::bad_alloc&) {
    delete m; set_error("hb_mesh_create: out of memory"); return HB_ERR_OOM;
  }
  *out = m;
  return HB_OK;
}

extern "C" int hb_mesh_sizes(const hb_mesh* m, hb_sizes* s) {
  if (!m || !s) { set_error("hb_mesh_sizes: null pointer"); return HB_ERR_ARG; }
  s->E_global = m->E_global;
  s->E_local = (int64_t)m->elems.size();
  s->N_L = s->E_local * m->NP3;
  s->N_G = m->NG;
  s->n_owned = (int64_t)m->owned.size();
  s->n_halo = (int64_t)m->halo.size();
  s->n_intA = m->nA; s->n_halo_elems = m->nH; s->n_intB = m->nB;
  s->n_neighbors = (int32_t)m->nbr.size();
  s->rank = m->rank; s->P = m->P;
  s->grid[0] = m->grid[0]; s->grid[1] = m->grid[1]; s->grid[2] = m->grid[2];
  return HB_OK;
}

#define HB_CHECK_PTR(p, name) \
  if (!(p)) { set_error(std::string(name) + ": null pointer"); return HB_ERR_ARG; }

extern "C" int hb_mesh_elements(const hb_mesh* m, int64_t* out) {
  HB_CHECK_PTR(m, "hb_mesh_elements"); HB_CHECK_PTR(out, "hb_mesh_elements");
  std::copy(m->elems.begin(), m->elems.end(), out);
  return HB_OK;
}

extern "C" int hb_mesh_l2g(const hb_mesh* m, int64_t* gid) {
  HB_CHECK_PTR(m, "hb_mesh_l2g"); HB_CHECK_PTR(gid, "hb_mesh_l2g");
  const int N = m->box.N, NP = m->NP, NP3 = m->NP3;
  const int64_t nx = m->box.nx, ny = m->box.ny;
  const int64_t gx = nx * N + 1, gy = ny * N + 1;
  for (size_t le = 0; le < m->elems.size(); ++le) {
    int64_t e = m->elems[le];
    int64_t ex = e % nx, ey = (e / nx) % ny, ez = e / (nx * ny);
    for (int k = 0; k < NP; ++k)
      for (int j = 0; j < NP; ++j)
        for (int i = 0; i < NP; ++i)
          gid[le * NP3 + i + NP * (j + NP * k)] = (ex * N + i) + gx * ((ey * N + j) + gy * (ez * N + k));
  }
  return HB_OK;
}

extern "C" int hb_mesh_local_index(const hb_mesh* m, int32_t* idx) {
  HB_CHECK_PTR(m, "hb_mesh_local_index"); HB_CHECK_PTR(idx, "hb_mesh_local_index");
  std::copy(m->idx.begin(), m->idx.end(), idx);
  return HB_OK;
}

extern "C" int hb_mesh_owned(const hb_mesh* m, int64_t* o) {
  HB_CHECK_PTR(m, "hb_mesh_owned"); HB_CHECK_PTR(o, "hb_mesh_owned");
  std::copy(m->owned.begin(), m->owned.end(), o);
  return HB_OK;
}

extern "C" int hb_mesh_halo(const hb_mesh* m, int64_t* h) {
  HB_CHECK_PTR(m, "hb_mesh_halo");
  if (!m->halo.empty()) { HB_CHECK_PTR(h, "hb_mesh_halo"); }
  std::copy(m->halo.begin(), m->halo.end(), h);
  return HB_OK;
}

extern "C" int hb_mesh_neighbors(const hb_mesh* m, int32_t* ranks, int64_t* sc, int64_t* rc) {
  HB_CHECK_PTR(m, "hb_mesh_neighbors");
  for (size_t t = 0; t < m->nbr.size(); ++t) {
    if (ranks) ranks[t] = m->nbr[t];
    if (sc) sc[t] = (int64_t)m->send_loc[t].size();
    if (rc) rc[t] = m->recv_cnt[t];
  }
  return HB_OK;
}

extern "C" int hb_mesh_send_list(const hb_mesh* m, int q, int64_t* gids) {
  HB_CHECK_PTR(m, "hb_mesh_send_list");
  if (q < 0 || q >= (int)m->nbr.size()) { set_error("hb_mesh_send_list: neighbour index out of range"); return HB_ERR_ARG; }
  if (!m->send_gid[q].empty()) { HB_CHECK_PTR(gids, "hb_mesh_send_list"); }
  std::copy(m->send_gid[q].begin(), m->send_gid[q].end(), gids);
  return HB_OK;
}

extern "C" int hb_mesh_geometry(const hb_mesh* m, double* G) {
  HB_CHECK_PTR(m, "hb_mesh_geometry"); HB_CHECK_PTR(G, "hb_mesh_geometry");
  const size_t n = m->elems.size() * (size_t)m->NP3;
  if (m->has_G) { std::copy(m->G_custom.begin(), m->G_custom.end(), G); return HB_OK; }
  // axis-aligned box elements: G_rr = w_i w_j w_k J (2/hx)^2 etc., cross terms 0
  const double hx = m->box.ext[0], hy = m->box.ext[1], hz = m->box.ext[2];
  const double J = hx * hy * hz / 8.0;
  const int NP = m->NP;
  for (size_t s = 0; s < n; ++s) {
    int nd = (int)(s % m->NP3);
    int i = nd % NP, j = (nd / NP) % NP, k = nd / (NP * NP);
    double wq = m->w[i] * m->w[j] * m->w[k] * J;
    double* g = G + 6 * s;
    g[0] = wq * (2.0 / hx) * (2.0 / hx); g[1] = 0.0; g[2] = 0.0;
    g[3] = wq * (2.0 / hy) * (2.0 / hy); g[4] = 0.0;
    g[5] = wq * (2.0 / hz) * (2.0 / hz);
  }
  return HB_OK;
}

extern "C" int hb_mesh_set_geometry(hb_mesh* m, const double* G) {
  HB_CHECK_PTR(m, "hb_mesh_set_geometry"); HB_CHECK_PTR(G, "hb_mesh_set_geometry");
  try {
    m->G_custom.assign(G, G + m->elems.size() * (size_t)m->NP3 * 6);
  } catch (const std::bad_alloc&) { set_error("hb_mesh_set_geometry: out of memory"); return HB_ERR_OOM; }
  m->has_G = true;
  return HB_OK;
}

extern "C" int hb_mesh_mass(const hb_mesh* m, double* M) {
  HB_CHECK_PTR(m, "hb_mesh_mass"); HB_CHECK_PTR(M, "hb_mesh_mass");
  const int N = m->box.N, NP = m->NP, NP3 = m->NP3;
  const int64_t nx = m->box.nx, ny = m->box.ny, nz = m->box.nz;
  if (m->box.mass_mode == 1) {
    if (m->has_B) { std::copy(m->B_custom.begin(), m->B_custom.end(), M); return HB_OK; }
    const double J = m->box.ext[0] * m->box.ext[1] * m->box.ext[2] / 8.0;
    for (size_t le = 0; le < m->elems.size(); ++le)
      for (int n = 0; n < NP3; ++n) {
        int i = n % NP, j = (n / NP) % NP, k = n / (NP * NP);
        M[le * NP3 + n] = m->w[i] * m->w[j] * m->w[k] * J;
      }
    return HB_OK;
  }
  // W = 1 / (number of elements sharing the point) (c1); per axis 2 on interior
  // element boundaries, 1 elsewhere.
  for (size_t le = 0; le < m->elems.size(); ++le) {
    int64_t e = m->elems[le];
    int64_t ex = e % nx, ey = (e / nx) % ny, ez = e / (nx * ny);
    for (int n = 0; n < NP3; ++n) {
      int i = n % NP, j = (n / NP) % NP, k = n / (NP * NP);
      auto cnt = [N](int64_t P0, int64_t nel) { return (P0 % N == 0 && P0 > 0 && P0 < nel * N) ? 2 : 1; };
      int c = cnt(ex * N + i, nx) * cnt(ey * N + j, ny) * cnt(ez * N + k, nz);
      M[le * NP3 + n] = 1.0 / c;
    }
  }
  return HB_OK;
}

extern "C" int hb_mesh_set_mass(hb_mesh* m, const double* M) {
  HB_CHECK_PTR(m, "hb_mesh_set_mass"); HB_CHECK_PTR(M, "hb_mesh_set_mass");
  if (m->box.mass_mode != 1) { set_error("hb_mesh_set_mass: only the mode-1 mass B can be overridden"); return HB_ERR_STATE; }
  try {
    m->B_custom.assign(M, M + m->elems.size() * (size_t)m->NP3);
  } catch (const std::bad_alloc&) { set_error("hb_mesh_set_mass: out of memory"); return HB_ERR_OOM; }
  m->has_B = true;
  return HB_OK;
}

extern "C" int hb_mesh_destroy(hb_mesh* m) {
  delete m;
  return HB_OK;
}
