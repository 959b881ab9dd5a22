"""Pins of the oracle's mapping / curl-interpolation node families (CPU only).

P:845 builds the isoparametric map on warp-and-blend nodes; reading R32 takes Warburton's
warp & blend with alpha = 0 (family 1) beside the equispaced lattice (family 0, R10).  What the
construction fixes, checked here against other sources than its own formula:
- the nodes on every edge are the Gauss-Lobatto-Legendre points (numpy's Legendre-derivative roots);
- the tetrahedron's nodes on every face are the triangle's node set (face restriction);
- the set is invariant under every permutation of the vertices (symmetry);
- for N <= 2 it is the lattice (the GLL points are equispaced there); family 0 is the lattice k/N;
- all nodes lie in the simplex, the set is unisolvent and its Lebesgue constant is far below the
  equispaced lattice's (the purpose of the construction);
- a curved mesh built on it preserves the free stream and conserves.
"""
import itertools
import math

import numpy as np
import pytest

import es_inputs as I
import oracle as O


def _gll(N):
    r = np.polynomial.legendre.Legendre.basis(N).deriv().roots()
    return np.sort(np.concatenate([[-1.0], np.real(r), [1.0]]))


def _key(lam, dec=11):
    return sorted(tuple(np.round(row, dec) + 0.0) for row in lam)


@pytest.mark.parametrize("d", [2, 3])
@pytest.mark.parametrize("N", [3, 4, 5, 6, 8, 9])
def test_edges_are_gll(d, N):
    if d == 2 and N == 9:
        N = 11  # the triangle's curl-free use goes to p + 1 = 11 for p = 10
    _, lam = O.nodes(d, N, 1)
    g = _gll(N)
    for i, j in itertools.combinations(range(d + 1), 2):
        others = [k for k in range(d + 1) if k not in (i, j)]
        on = np.all(np.abs(lam[:, others]) < 1e-15, axis=1)
        r = np.sort(lam[on, j] - lam[on, i])
        assert len(r) == N + 1
        assert np.abs(r - g).max() < 2e-15, (i, j, np.abs(r - g).max())


@pytest.mark.parametrize("N", [3, 4, 6, 8, 9])
def test_tet_faces_are_triangle_nodes(N):
    _, l3 = O.nodes(3, N, 1)
    _, l2 = O.nodes(2, N, 1)
    for a in range(4):
        on = np.abs(l3[:, a]) < 1e-15
        face = l3[on][:, [k for k in range(4) if k != a]]
        assert face.shape == l2.shape
        assert _key(face) == _key(l2)


@pytest.mark.parametrize("d,N", [(2, 5), (2, 8), (2, 10), (3, 5), (3, 8), (3, 9)])
def test_vertex_permutation_symmetry(d, N):
    _, lam = O.nodes(d, N, 1)
    ref = _key(lam)
    for perm in itertools.permutations(range(d + 1)):
        assert _key(lam[:, list(perm)]) == ref


@pytest.mark.parametrize("d", [2, 3])
def test_low_degree_and_family0_are_lattice(d):
    for N in (1, 2, 3, 6):
        xi0, lam0 = O.nodes(d, N, 0)
        assert np.abs(lam0 * N - np.round(lam0 * N)).max() < 1e-14
        assert np.abs(xi0 - (-1 + 2 * lam0[:, 1:])).max() < 1e-15
        if N <= 2:
            xi1, lam1 = O.nodes(d, N, 1)
            assert np.abs(lam1 - lam0).max() < 1e-15


def _monomials(x, N):
    d = x.shape[1]
    cols = []
    for e in itertools.product(range(N + 1), repeat=d):
        if sum(e) <= N:
            cols.append(np.prod([x[:, k] ** e[k] for k in range(d)], axis=0))
    return np.stack(cols, axis=1)


def _lebesgue(d, N, family, ns):
    _, lam = O.nodes(d, N, family)
    x = lam[:, 1:]
    V = _monomials(x, N)
    # sample points of the simplex (a fine lattice)
    pts = [np.array(c) / ns for c in itertools.product(range(ns + 1), repeat=d) if sum(c) <= ns]
    P = _monomials(np.array(pts), N)
    Lg = np.linalg.solve(V.T, P.T)  # Lagrange basis values [M][npts]
    return np.abs(Lg).sum(axis=0).max(), np.linalg.cond(V)


@pytest.mark.parametrize("d,N,ns", [(2, 8, 60), (2, 10, 60), (3, 6, 24), (3, 8, 24)])
def test_inside_unisolvent_and_lebesgue(d, N, ns):
    _, lam = O.nodes(d, N, 1)
    assert lam.min() >= 0.0 and np.abs(lam.sum(axis=1) - 1).max() < 1e-15
    leb1, cond = _lebesgue(d, N, 1, ns)
    leb0, _ = _lebesgue(d, N, 0, ns)
    assert cond < 1e12  # unisolvent
    assert leb1 < 0.6 * leb0, (leb1, leb0)  # 2D N = 8: 5.6 vs 23.6; 3D N = 8: 13.7 vs 40.3


@pytest.mark.parametrize("d,p", [(2, 4), (3, 3)])
def test_warp_and_blend_mesh_free_stream_conservation_entropy(d, p):
    L = 2.0 if d == 2 else 2 * math.pi
    mesh = I.split_cartesian(d, 3, L)
    om = O.Mesh(mesh, p, warp=I.paper_warp(d, L), nodes=1)
    om0 = O.Mesh(mesh, p, warp=I.paper_warp(d, L), nodes=0)
    # another node family interpolates the same warp by another degree-p map
    assert np.abs(om.geometry(4)["Jt"] - om0.geometry(4)["Jt"]).max() > 1e-8
    # free stream
    u = om.project(I.free_stream(om.node_coords(), d))
    du, _ = om.rhs(u, flux_mode=1, variant=0)
    scale = max(np.abs(om.geometry(e)["G"]).max() / om.geometry(e)["Jt"].min() for e in range(om.ne))
    assert np.abs(du).max() < 1e-13 * scale * (p + 1) ** 2
    # conservation and the entropy balance on the periodic mesh
    xq = om.node_coords()
    u0 = I.density_wave(xq, L) if d == 2 else I.taylor_green(xq, Ma=0.3)
    u = I.perturb_modal(om.project(u0), d, p, seed=1, amp=2e-2)
    for fm in (0, 1):
        ref, st = om.rhs(u, flux_mode=fm, variant=0)
        assert np.abs(st.conservation[:d + 2]).max() < 1e-13 * np.abs(ref).max() * om.ne
        if fm == 0:
            assert abs(st.entropy_rate) < 1e-12 * st.entropy_abs
        else:
            assert st.entropy_rate < -1e-6 * st.entropy_abs
