"""Pins of the oracle's modal (compressed) metric storage -- CPU only.

The metric terms are polynomials of degree <= p in the reference coordinates (2D exact metrics of the
degree-p map: degree p - 1; 3D conservative curl form of the degree-(q+1) interpolant:
degree q = p), so with M = V^T W V = I the stored PKD coefficients g~ = V^T W G
reproduce G at the volume nodes, and the RHS on the reconstructed metrics equals the nodal one up
to rounding.  Pinned here by what the mathematics fixes:
- affine elements: g~ has only the constant mode, g~_0 = adj(A) sqrt(|ref|) (closed form);
- 2D curved: the coefficients of total degree p vanish (the metric has degree p - 1), while lower
  ones do not (the pin is not vacuous);
- 3D curved: V g~ = G at the volume nodes (the curl metric has degree <= q);
- the full RHS with modal metrics equals the nodal-metric RHS (2D and 3D, curved, ES flux).
"""
import math

import numpy as np
import pytest

import es_inputs as I
import oracle as O


def _mesh(d, M, p, warp, modal=0):
    L = 2.0 if d == 2 else 2 * math.pi
    mesh = I.split_cartesian(d, M, L)
    w = I.paper_warp(d, L) if warp else None
    return mesh, O.Mesh(mesh, p, warp=w, metric_storage=modal)


@pytest.mark.parametrize("d,p", [(2, 3), (3, 2), (3, 3)])
def test_affine_metric_is_constant_mode(d, p):
    mesh, om = _mesh(d, 3, p, warp=False)
    ref = I.reference_measure(d)
    for e in (0, 3, om.ne - 1):
        X = mesh["elem_vertex_coords"][e]
        A = ((X[1:] - X[0]) / 2.0).T
        adj = np.linalg.det(A) * np.linalg.inv(A)
        gm = om.metric_modal(e)
        assert np.abs(gm[:, 0] - adj.reshape(-1) * math.sqrt(ref)).max() < 1e-13 * np.abs(adj).max()
        assert np.abs(gm[:, 1:]).max() < 1e-13 * np.abs(adj).max()


@pytest.mark.parametrize("p", [2, 3, 4])
def test_2d_curved_metric_has_degree_p_minus_1(p):
    _, om = _mesh(2, 3, p, warp=True)
    deg = I.multi_index_degrees(2, p)
    assert len(deg) == om.Np
    top = deg == p
    low = (deg > 0) & (deg < p)
    big = 0.0
    for e in range(om.ne):
        gm = om.metric_modal(e)
        sc = np.abs(gm).max()
        assert np.abs(gm[:, top]).max() < 1e-12 * sc, e
        big = max(big, np.abs(gm[:, low]).max() / sc)
    assert big > 1e-3  # the warp really curves the elements


@pytest.mark.parametrize("p", [2, 3])
def test_3d_curl_metric_reconstructed_exactly(p):
    _, om = _mesh(3, 3, p, warp=True)
    V = O.ref_get(3, p, "V")
    worst, curved = 0.0, 0.0
    for e in range(om.ne):
        G = om.geometry(e)["G"].reshape(om.Nq, 9)
        gm = om.metric_modal(e)
        worst = max(worst, np.abs(V @ gm.T - G).max() / np.abs(G).max())
        curved = max(curved, np.abs(gm[:, 1:]).max() / np.abs(gm).max())
    assert worst < 1e-12
    assert curved > 1e-3


@pytest.mark.parametrize("d,p", [(2, 3), (3, 2), (3, 3)])
def test_rhs_with_modal_metrics_equals_nodal(d, p):
    mesh, om = _mesh(d, 3, p, warp=True)
    _, omm = _mesh(d, 3, p, warp=True, modal=1)
    x = om.node_coords()
    u = om.project(I.taylor_green(x) if d == 3 else I.density_wave(x))
    u = I.perturb_modal(u, d, p, seed=3)
    du, _ = om.rhs(u, flux_mode=1)
    dm, _ = omm.rhs(u, flux_mode=1)
    assert np.abs(dm - du).max() < 1e-11 * np.abs(du).max()
