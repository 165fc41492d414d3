// Internal declarations shared by the host mesher (mesh.cpp) and the device side (op.cu).
// Not part of the ABI; see include/hipbone_b200.h.
#pragma once

#include <cstdint>
#include <string>
#include <vector>

#include "../../include/hipbone_b200.h"

namespace hb {

void set_error(const std::string& msg);

// splitmix64 (c9, c12): z += 0x9E3779B97F4A7C15; z = (z^z>>30)*0xBF58476D1CE4E5B9;
// z = (z^z>>27)*0x94D049BB133111EB; return z^z>>31.
inline uint64_t splitmix64(uint64_t z) {
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

// 1-D basis: GLL nodes/weights by Newton on P_N', D by the closed form
// D_ij = P_N(x_i) / (P_N(x_j) (x_i - x_j)) (i != j), D_00 = -N(N+1)/4, D_NN = N(N+1)/4.
void gll_basis(int N, std::vector<double>& x, std::vector<double>& w, std::vector<double>& D);

}  // namespace hb

struct hb_mesh {
  hb_box box{};
  int P = 1, rank = 0;
  int grid[3] = {1, 1, 1};
  uint64_t seed = 0;
  int NP = 0, NP3 = 0;
  int64_t E_global = 0, NG = 0;
  std::vector<int64_t> elems;  // global element ids, local order [A | halo | B]
  int64_t nA = 0, nH = 0, nB = 0;
  std::vector<int32_t> idx;    // [E_local][NP3] local index into [owned | halo]
  std::vector<int64_t> owned;  // gids ascending
  std::vector<int64_t> halo;   // gids grouped by owner rank, then gid ascending
  std::vector<int32_t> nbr;    // neighbour ranks ascending
  std::vector<std::vector<int32_t>> send_loc;  // per neighbour: owned local indices to send
  std::vector<std::vector<int64_t>> send_gid;  // per neighbour: the same as gids
  std::vector<int64_t> recv_off, recv_cnt;     // per neighbour: segment of the halo part
  std::vector<double> x, w, D;                 // GLL basis
  bool has_G = false, has_B = false;
  std::vector<double> G_custom;  // [E_local][NP3][6] packed (paper layout)
  std::vector<double> B_custom;  // [E_local][NP3]
};
