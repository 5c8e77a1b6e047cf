// Partition plan of a conforming multi-patch domain for the subdomain (patch-per-GPU) mode
// (include/genalpha.h ga_partition_plan).  Host only.
//
// Gluing follows P:654-689: the global index map identifies two local basis functions iff they
// coincide on the interface, which for conforming patches with matching knot vectors (P:645-652,
// Assumption "conformity") means bitwise-equal control points.  A face is an interface iff its
// control-point set equals a face of another patch; a function is Dirichlet iff one of its copies
// lies on a face that is not an interface (homogeneous Dirichlet data on the boundary).
#include <algorithm>
#include <array>
#include <cstdint>
#include <cstring>
#include <map>
#include <vector>

#include "../../include/genalpha.h"

namespace {

using Key = std::array<uint64_t, 3>;

Key point_key(const double* x, int dim) {
  Key k = {0, 0, 0};
  for (int d = 0; d < dim; ++d) {
    double v = x[d];
    if (v == 0.0) v = 0.0;  // -0.0 and +0.0 are the same point
    memcpy(&k[d], &v, sizeof(double));
  }
  return k;
}

}  // namespace

extern "C" ga_status ga_partition_plan(int dim, int p, int n, int npatch, const double* const* ctrl,
                                       unsigned char* free_mask, unsigned char* owned, long long* iface,
                                       long long* n_iface, long long* n_free_global) {
  if ((dim != 2 && dim != 3) || p < 1 || n < 1 || npatch < 1 || !ctrl || !free_mask || !owned || !iface)
    return GA_ERR_ARG;
  for (int r = 0; r < npatch; ++r)
    if (!ctrl[r]) return GA_ERR_ARG;
  const int m = n + p;
  const long long mp = dim == 3 ? (long long)m * m * m : (long long)m * m;
  // global numbering by coincident control points
  std::map<Key, long long> id_of;
  std::vector<long long> gid((size_t)npatch * mp);
  for (int r = 0; r < npatch; ++r)
    for (long long i = 0; i < mp; ++i) {
      const Key k = point_key(ctrl[r] + i * dim, dim);
      auto it = id_of.find(k);
      long long g;
      if (it == id_of.end()) {
        g = (long long)id_of.size();
        id_of.emplace(k, g);
      } else {
        g = it->second;
      }
      gid[(size_t)r * mp + i] = g;
    }
  const long long nglob = (long long)id_of.size();
  // faces: (patch, axis, side) -> sorted global ids
  struct Face { int r, a, side; std::vector<long long> ids; std::vector<long long> loc; };
  std::vector<Face> faces;
  for (int r = 0; r < npatch; ++r)
    for (int a = 0; a < dim; ++a)
      for (int side = 0; side < 2; ++side) {
        Face f;
        f.r = r; f.a = a; f.side = side;
        const int want = side ? m - 1 : 0;
        for (long long i = 0; i < mp; ++i) {
          const long long li[3] = {i % m, (i / m) % m, dim == 3 ? i / ((long long)m * m) : 0};
          if (li[a] == want) {
            f.loc.push_back(i);
            f.ids.push_back(gid[(size_t)r * mp + i]);
          }
        }
        std::sort(f.ids.begin(), f.ids.end());
        faces.push_back(std::move(f));
      }
  std::map<std::vector<long long>, std::vector<int>> by_set;
  for (size_t fi = 0; fi < faces.size(); ++fi) by_set[faces[fi].ids].push_back((int)fi);
  std::vector<char> dirichlet((size_t)nglob, 0);
  for (size_t fi = 0; fi < faces.size(); ++fi) {
    const Face& f = faces[fi];
    bool matched = false;
    for (int o : by_set[f.ids])
      if (faces[o].r != f.r) matched = true;
    if (!matched) {
      // a face sharing some but not all points with a face of another patch is non-conforming
      for (size_t oi = 0; oi < faces.size(); ++oi) {
        const Face& g = faces[oi];
        if (g.r == f.r) continue;
        std::vector<long long> common;
        std::set_intersection(f.ids.begin(), f.ids.end(), g.ids.begin(), g.ids.end(), std::back_inserter(common));
        // faces of conforming neighbours that are not glued share at most a vertex (2D) or an
        // edge line of m points (3D)
        const size_t most = dim == 2 ? 1 : (size_t)m;
        if (common.size() > most) return GA_ERR_CONFORMITY;
      }
      for (long long g : f.ids) dirichlet[(size_t)g] = 1;
    }
  }
  // copies, owners, interface slots (first-copy order)
  std::vector<int> copies((size_t)nglob, 0);
  for (long long g : gid) copies[(size_t)g] += 1;
  std::vector<char> seen((size_t)nglob, 0);
  std::vector<long long> slot((size_t)nglob, -1);
  long long nif = 0, nfree = 0;
  for (int r = 0; r < npatch; ++r)
    for (long long i = 0; i < mp; ++i) {
      const size_t e = (size_t)r * mp + i;
      const long long g = gid[e];
      const bool fr = !dirichlet[(size_t)g];
      free_mask[e] = fr ? 1 : 0;
      owned[e] = 0;
      iface[e] = -1;
      if (!fr) continue;
      if (!seen[(size_t)g]) {
        seen[(size_t)g] = 1;
        owned[e] = 1;
        ++nfree;
        if (copies[(size_t)g] >= 2) slot[(size_t)g] = nif++;
      }
      iface[e] = slot[(size_t)g];
    }
  if (n_iface) *n_iface = nif;
  if (n_free_global) *n_free_global = nfree;
  return GA_OK;
}
