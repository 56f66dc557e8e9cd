// hex_dofs.cpp -- DoF numbering of a conforming unstructured hex mesh (host; the
// DoF-handler step of PAPER.md P:694-705 §3.1; R21).
//
// Continuous Q_k on the GLL nodes: one DoF per vertex, k-1 per edge, (k-1)^2 per
// face, (k-1)^3 per cell interior.  Two cells that share an edge or a face may see it
// in different local orientations; the DoFs of an edge / face are therefore laid out in
// a frame fixed by the GLOBAL vertex numbers alone:
//   edge {a, b}: position p = 0..k-2 counted from the smaller vertex number;
//   face {v0..v3}: origin = smallest vertex number, first axis towards the smaller of
//   the origin's two face neighbours; interior node (a, b), a, b = 1..k-1, gets
//   (a - 1) + (b - 1)(k - 1).
// The GLL nodes are symmetric in [0,1], so both cells' support points agree.
#include <algorithm>
#include <array>
#include <climits>
#include <cstdint>
#include <string>
#include <unordered_map>
#include <vector>

#include "internal.h"

namespace mf {

namespace {

struct FaceHash {
  size_t operator()(const std::array<int32_t, 4> &a) const {
    uint64_t h = 1469598103934665603ull;
    for (int32_t v : a) h = (h ^ (uint32_t)v) * 1099511628211ull;
    return (size_t)h;
  }
};

struct FaceRec {
  int64_t base = -1;
  int count = 0;
};

// local vertex of the reference corner (a, b, c), a, b, c in {0, 1}
inline int lv(int a, int b, int c) { return a + 2 * b + 4 * c; }

}  // namespace

mf_status hex_number_dofs(int k, int64_t n_cells, const int32_t *CV, int32_t *cell_dofs, int64_t *n_dofs,
                          uint8_t *is_boundary, int64_t capacity, std::string *err) {
  const int N = k + 1, NV = N * N * N, km = k - 1;
  std::unordered_map<int32_t, int64_t> vdof;
  std::unordered_map<uint64_t, int64_t> edof;
  std::unordered_map<std::array<int32_t, 4>, FaceRec, FaceHash> faces;
  int64_t next = 0;
  // pass 1: face multiplicities (manifold / conformity check, boundary faces)
  for (int64_t c = 0; c < n_cells; ++c) {
    const int32_t *v = CV + 8 * c;
    for (int a = 0; a < 8; ++a)
      for (int b = a + 1; b < 8; ++b)
        if (v[a] == v[b]) {
          *err = "cell " + std::to_string(c) + " repeats a vertex";
          return MF_ERR_ARGUMENT;
        }
    for (int d = 0; d < 3; ++d)
      for (int side = 0; side < 2; ++side) {
        std::array<int32_t, 4> key;
        int m = 0;
        for (int j = 0; j < 8; ++j)
          if (((j >> d) & 1) == side) key[m++] = v[j];
        std::sort(key.begin(), key.end());
        if (++faces[key].count > 2) {
          *err = "a face is shared by more than two cells (non-conforming or non-manifold mesh)";
          return MF_ERR_ARGUMENT;
        }
      }
  }
  // pass 2: number in order of first appearance
  for (int64_t c = 0; c < n_cells; ++c) {
    const int32_t *v = CV + 8 * c;
    int64_t interior = -1;
    for (int i = 0; i < NV; ++i) {
      const int id[3] = {i % N, (i / N) % N, i / (N * N)};
      int nb = 0;
      for (int d = 0; d < 3; ++d) nb += (id[d] == 0 || id[d] == k);
      int64_t dof = -1;
      if (nb == 3) {
        const int32_t gv = v[lv(id[0] / k, id[1] / k, id[2] / k)];
        auto it = vdof.find(gv);
        if (it == vdof.end()) it = vdof.emplace(gv, next++).first;
        dof = it->second;
      } else if (nb == 2) {
        int f = 0;
        while (id[f] == 0 || id[f] == k) ++f;  // the free axis (interior coordinate)
        int ca[3], cb[3];
        for (int d = 0; d < 3; ++d) ca[d] = cb[d] = id[d] / k;
        ca[f] = 0;
        cb[f] = 1;
        const int32_t ga = v[lv(ca[0], ca[1], ca[2])], gb = v[lv(cb[0], cb[1], cb[2])];
        const uint64_t key = ((uint64_t)(uint32_t)std::min(ga, gb) << 32) | (uint32_t)std::max(ga, gb);
        auto it = edof.find(key);
        if (it == edof.end()) {
          it = edof.emplace(key, next).first;
          next += km;
        }
        const int t = id[f];
        dof = it->second + (ga < gb ? t - 1 : k - t - 1);
      } else if (nb == 1) {
        int d = 0;
        while (id[d] != 0 && id[d] != k) ++d;  // the fixed axis
        const int u = d == 0 ? 1 : 0, w = d == 2 ? 1 : 2;
        int32_t cg[2][2];
        std::array<int32_t, 4> key;
        for (int pu = 0; pu < 2; ++pu)
          for (int pw = 0; pw < 2; ++pw) {
            int cc[3];
            cc[d] = id[d] / k;
            cc[u] = pu;
            cc[w] = pw;
            cg[pu][pw] = v[lv(cc[0], cc[1], cc[2])];
            key[2 * pu + pw] = cg[pu][pw];
          }
        std::sort(key.begin(), key.end());
        FaceRec &fr = faces[key];
        if (fr.base < 0) {
          fr.base = next;
          next += (int64_t)km * km;
        }
        int ou = 0, ow = 0;
        for (int pu = 0; pu < 2; ++pu)
          for (int pw = 0; pw < 2; ++pw)
            if (cg[pu][pw] < cg[ou][ow]) {
              ou = pu;
              ow = pw;
            }
        const bool first_u = cg[1 - ou][ow] < cg[ou][1 - ow];
        const int du = ou == 0 ? id[u] : k - id[u], dw = ow == 0 ? id[w] : k - id[w];
        const int a = first_u ? du : dw, b = first_u ? dw : du;
        dof = fr.base + (a - 1) + (int64_t)(b - 1) * km;
      } else {
        if (interior < 0) {
          interior = next;
          next += (int64_t)km * km * km;
        }
        dof = interior + (id[0] - 1) + (int64_t)km * ((id[1] - 1) + (int64_t)km * (id[2] - 1));
      }
      cell_dofs[c * NV + i] = (int32_t)dof;
    }
    if (next > INT32_MAX) {
      *err = "more than 2^31 - 1 DoFs";
      return MF_ERR_ARGUMENT;
    }
  }
  *n_dofs = next;
  if (is_boundary) {
    if (next > capacity) {
      *err = "is_boundary capacity < n_dofs";
      return MF_ERR_LENGTH;
    }
    std::fill(is_boundary, is_boundary + next, (uint8_t)0);
    for (int64_t c = 0; c < n_cells; ++c) {
      const int32_t *v = CV + 8 * c;
      for (int d = 0; d < 3; ++d)
        for (int side = 0; side < 2; ++side) {
          std::array<int32_t, 4> key;
          int m = 0;
          for (int j = 0; j < 8; ++j)
            if (((j >> d) & 1) == side) key[m++] = v[j];
          std::sort(key.begin(), key.end());
          if (faces[key].count != 1) continue;
          for (int i = 0; i < NV; ++i) {
            const int id[3] = {i % N, (i / N) % N, i / (N * N)};
            if (id[d] == side * k) is_boundary[cell_dofs[c * NV + i]] = 1;
          }
        }
    }
  }
  return MF_OK;
}

}  // namespace mf
