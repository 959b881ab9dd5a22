// mesh_plan.cpp -- connectivity, orientation permutations (R11) and the
// element-partition / face-halo plan.  Host C++, product code.
#include <algorithm>
#include <array>
#include <unordered_map>

#include "internal.h"

namespace esb {
namespace {

// facet -> local vertices in (eta_f1 start, eta_f1 end, collapse) order, from the facet node
// parametrisations P:208-212 (triangle) and P:271-273 (tetrahedron, corrected map R1)
const int kTriFace[3][2] = {{0, 1}, {1, 2}, {0, 2}};
const int kTetFace[4][3] = {{0, 1, 3}, {1, 2, 3}, {0, 2, 3}, {0, 1, 2}};

struct Key {
  std::array<int64_t, 3> v;
  bool operator==(const Key& o) const { return v == o.v; }
};
struct KeyHash {
  size_t operator()(const Key& k) const {
    uint64_t h = 1469598103934665603ull;
    for (int64_t x : k.v) {
      h ^= (uint64_t)x + 0x9e3779b97f4a7c15ull + (h << 6) + (h >> 2);
      h *= 1099511628211ull;
    }
    return (size_t)h;
  }
};

}  // namespace

bool build_mesh_plan(int d, int64_t ne, const int64_t* ev, int rank, int world, MeshPlan& plan,
                     std::string& err) {
  int nv = d + 1, Nf = d + 1;
  plan.d = d;
  plan.Nf = Nf;
  plan.ne = ne;
  plan.nbr.assign(ne * Nf, -1);
  plan.nbr_face.assign(ne * Nf, -1);
  plan.reflect.assign(ne * Nf, 0);
  std::unordered_map<Key, int64_t, KeyHash> first;  // face key -> e*Nf+z of the first visitor
  first.reserve((size_t)(ne * Nf / 2 + 16));
  auto fv = [&](int z, int k) { return d == 2 ? kTriFace[z][k] : kTetFace[z][k]; };
  for (int64_t e = 0; e < ne; ++e) {
    const int64_t* v = ev + e * nv;
    for (int i = 0; i < nv; ++i)
      for (int j = i + 1; j < nv; ++j)
        if (v[i] == v[j]) {
          err = "element " + std::to_string(e) + " repeats a vertex id (need M >= 3)";
          return false;
        }
    for (int z = 0; z < Nf; ++z) {
      Key k{{-1, -1, -1}};
      for (int t = 0; t < d; ++t) k.v[t] = v[fv(z, t)];
      std::sort(k.v.begin(), k.v.begin() + d);
      auto it = first.find(k);
      if (it == first.end()) {
        first.emplace(k, e * Nf + z);
        continue;
      }
      int64_t o = it->second / Nf;
      int zo = (int)(it->second % Nf);
      if (plan.nbr[o * Nf + zo] >= 0) {
        err = "face shared by more than two elements";
        return false;
      }
      const int64_t* w = ev + o * nv;
      // same collapse vertex on both sides (3D), start/end equal or swapped
      if (d == 3 && v[fv(z, 2)] != w[fv(zo, 2)]) {
        err = "collapse vertices differ on face (element " + std::to_string(e) + ")";
        return false;
      }
      int64_t a0 = v[fv(z, 0)], a1 = v[fv(z, 1)], b0 = w[fv(zo, 0)], b1 = w[fv(zo, 1)];
      int refl;
      if (a0 == b0 && a1 == b1)
        refl = 0;
      else if (a0 == b1 && a1 == b0)
        refl = 1;
      else {
        err = "inconsistent face orientation";
        return false;
      }
      plan.nbr[e * Nf + z] = o;
      plan.nbr_face[e * Nf + z] = zo;
      plan.reflect[e * Nf + z] = refl;
      plan.nbr[o * Nf + zo] = e;
      plan.nbr_face[o * Nf + zo] = z;
      plan.reflect[o * Nf + zo] = refl;
    }
  }
  for (int64_t i = 0; i < ne * Nf; ++i)
    if (plan.nbr[i] < 0) {
      err = "unmatched face (mesh must be closed / periodic)";
      return false;
    }
  // ---------------- partition: contiguous element ranges ----------------
  int64_t first_el, nloc;
  rank_range(ne, rank, world, first_el, nloc);
  plan.first = first_el;
  plan.nloc = nloc;
  auto owner = [&](int64_t g) {
    // inverse of rank_range: the rank r with first(r) <= g < first(r+1)
    int64_t r = (g * world) / ne;
    while (r > 0 && ne * r / world > g) --r;
    while (r + 1 < world && ne * (r + 1) / world <= g) ++r;
    return (int)r;
  };
  plan.face_slot.assign(nloc * Nf, -1);
  plan.face_reflect.assign(nloc * Nf, 0);
  // faces this rank needs from rank s: remote (element, face) pairs sorted by (element, face)
  std::vector<std::vector<int64_t>> need(world), give(world);
  for (int64_t k = 0; k < nloc; ++k) {
    int64_t e = first_el + k;
    bool remote = false;
    for (int z = 0; z < Nf; ++z) {
      int64_t o = plan.nbr[e * Nf + z];
      int r = owner(o);
      plan.face_reflect[k * Nf + z] = plan.reflect[e * Nf + z];
      if (r == rank) {
        plan.face_slot[k * Nf + z] = (o - first_el) * Nf + plan.nbr_face[e * Nf + z];
      } else {
        remote = true;
        need[r].push_back(o * Nf + plan.nbr_face[e * Nf + z]);
        give[r].push_back(e * Nf + z);  // the neighbour needs our trace of this face
      }
    }
    (remote ? plan.boundary : plan.interior).push_back(k);
  }
  plan.send_count.assign(world, 0);
  plan.send_offset.assign(world, 0);
  plan.recv_count.assign(world, 0);
  plan.recv_offset.assign(world, 0);
  plan.send_slots.clear();
  int64_t halo_base = nloc * Nf, off = 0, soff = 0;
  std::unordered_map<int64_t, int64_t> halo_index;
  for (int r = 0; r < world; ++r) {
    std::sort(need[r].begin(), need[r].end());
    std::sort(give[r].begin(), give[r].end());
    plan.recv_offset[r] = off;
    plan.recv_count[r] = (int64_t)need[r].size();
    for (size_t i = 0; i < need[r].size(); ++i) halo_index[need[r][i]] = halo_base + off + (int64_t)i;
    off += (int64_t)need[r].size();
    plan.send_offset[r] = soff;
    plan.send_count[r] = (int64_t)give[r].size();
    for (int64_t gf : give[r]) plan.send_slots.push_back((gf / Nf - first_el) * Nf + gf % Nf);
    soff += (int64_t)give[r].size();
  }
  plan.n_halo = off;
  for (int64_t k = 0; k < nloc; ++k) {
    int64_t e = first_el + k;
    for (int z = 0; z < Nf; ++z)
      if (plan.face_slot[k * Nf + z] < 0)
        plan.face_slot[k * Nf + z] = halo_index.at(plan.nbr[e * Nf + z] * Nf + plan.nbr_face[e * Nf + z]);
  }
  return true;
}

}  // namespace esb
