// internal.h -- shared declarations of the B200 library (host setup <-> device kernels <-> ABI).
// Product code; shares nothing with oracle/.
#pragma once
#include <cstdint>
#include <string>
#include <vector>

namespace esb {

// ----------------------------------------------------------------------------------------------
// Host-built reference tables for one (dim, p), q = p.  Everything the kernels need about
// the reference element is here; it is re-derived for the line structure of the operators:
//   S^(l) = (Q^(l) - Q^(l)^T)/2 restricted to an eta_k line = c_k(line) * skew(X_{k,l}),
// with X one of the 1D matrices below.
// ----------------------------------------------------------------------------------------------
struct RefTables {
  int d = 0, p = 0, n = 0, Nq = 0, Nf = 0, Nqf = 0, Np = 0;
  std::vector<double> eta, w;    // Legendre-Gauss nodes / weights (n)
  std::vector<double> eta3, w3;  // Gauss-Jacobi (1,0) nodes / weights (n), tet eta3 direction
  // 1D skew-symmetric line operators, row-major n x n
  std::vector<double> skQ1;  // skew(diag(w) D)
  std::vector<double> skA1;  // skew(diag(w (1+eta)/2) D)
  std::vector<double> skA2;  // skew(diag(w (1-eta)/2) D)
  std::vector<double> skA3;  // skew(diag(w (1-eta^2)/4) D)            (tet)
  std::vector<double> skA4;  // skew(diag(w3 (1-eta3)) D3)              (tet)
  std::vector<double> fQ1, fA1, fA2, fA3, fA4;  // the unskewed X (Q^(l) line blocks, linear advection)
  std::vector<double> lL, lR;    // LG Lagrange basis at -1 and +1 (n)
  std::vector<double> l3L;       // GJ(1,0) Lagrange basis at -1 (n)       (tet)
  std::vector<double> lint4;     // [j][b] LG basis l_b at eta3_j         (tet facet 4)
  // PKD sum-factorisation tables: psi1[a1][a], psi2[a1][a2][b], psi3[s][a3][c]
  std::vector<double> psi1, psi2, psi3;
  std::vector<int> pair_a1, pair_a2, pair_off;  // (a1,a2) pairs (tet) / a1 rows (tri): first mode
  std::vector<double> Wvol;      // [Nq] volume weights (P:205 / P:267)
  std::vector<double> Bf;        // [Nf][Nqf] facet weights (P:211 / P:281)
  std::vector<double> nhat;      // [Nf][3] reference outward normals
  std::vector<double> xi_vol;    // [Nq][d] reference coordinates of volume nodes
  std::vector<double> xi_face;   // [Nf][Nqf][d]
  // geometry interpolation (lattice of degree p for the map, q+1 for curl metrics, R10)
  int Npg = 0, Ncl = 0;
  int nodes = 0;                 // node family of the map and the curl interpolant (0 lattice R10, 1 warp & blend R32)
  std::vector<double> lat_bary;  // [Npg][d+1] barycentric coordinates of mapping nodes
  std::vector<double> LmapV;     // [Nq][Npg]   Lagrange basis of the map at volume nodes
  std::vector<double> DmapV;     // [d][Nq][Npg] gradients at volume nodes (2D metrics)
  std::vector<double> DmapF;     // [d][Nf*Nqf][Npg] gradients at facet nodes (2D)
  std::vector<double> DmapM;     // [d][Npg][Npg] gradients at the mapping nodes (J for J~)
  std::vector<double> LmapC;     // [Ncl][Npg] map basis at curl-lattice nodes (3D)
  std::vector<double> DmapC;     // [d][Ncl][Npg]
  std::vector<double> DcurlV;    // [d][Nq][Ncl] curl-lattice basis gradients at volume nodes
  std::vector<double> DcurlF;    // [d][Nf*Nqf][Ncl]
};

bool build_ref_tables(int d, int p, RefTables& t, std::string& err, int nodes = 0);
// barycentric coordinates [M][d+1] of the degree-N mapping node family (0 lattice, 1 warp & blend)
std::vector<double> node_family_bary(int d, int N, int family);
// dense S^(l) [l][j][i] and (R^(z)T B) [z][f][i] for the brute-force ablation (volume_mode 2)
void build_dense_tables(const RefTables& t, std::vector<double>& S, std::vector<double>& RB);
// PKD basis, mapping Lagrange basis and its reference gradients at arbitrary points (es_eval_points)
bool eval_point_tables(int d, int p, const double* xi, int npts, std::vector<double>& pkd, std::vector<double>& lmap,
                       std::vector<double>& dmap, int nodes = 0);

// ----------------------------------------------------------------------------------------------
// Host mesh plan: connectivity with the orientation rule R11, and the partition/halo
// plan for `world` ranks (contiguous element ranges).
// ----------------------------------------------------------------------------------------------
struct MeshPlan {
  int d = 0, Nf = 0;
  int64_t ne = 0, first = 0, nloc = 0;
  std::vector<int64_t> nbr;      // [ne_global][Nf] neighbour element
  std::vector<int> nbr_face;     // [ne_global][Nf]
  std::vector<int> reflect;      // [ne_global][Nf] 1 = eta_f1 reversed on the neighbour
  // local view
  std::vector<int64_t> face_slot;  // [nloc][Nf] trace slot of the neighbour face (local or halo)
  std::vector<int> face_reflect;   // [nloc][Nf]
  std::vector<int64_t> send_slots; // local trace slots to send, grouped by destination rank
  std::vector<int64_t> send_count, send_offset;  // [world]
  std::vector<int64_t> recv_count, recv_offset;  // [world] halo faces received from each rank
  int64_t n_halo = 0;
  std::vector<int64_t> interior, boundary;  // local element ids without / with remote neighbours
};

bool build_mesh_plan(int d, int64_t ne, const int64_t* ev, int rank, int world, MeshPlan& plan,
                     std::string& err);

// per-element strides of the device arrays, rounded up to an even number of doubles so that every
// element block is 16-byte aligned for bulk (TMA) copies
inline int even_up(int x) { return (x + 1) & ~1; }

// element range of a rank
inline void rank_range(int64_t ne, int rank, int world, int64_t& first, int64_t& count) {
  first = ne * rank / world;
  count = ne * (rank + 1) / world - first;
}

}  // namespace esb
