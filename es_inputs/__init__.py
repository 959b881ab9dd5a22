"""Seeded synthetic inputs shared by the oracle and the CUDA path (no method arithmetic here).

Everything in this module is *input*: meshes, the geometry warp (the user map), initial states in
conservative variables, and seeded perturbations of modal coefficient arrays.  Nothing here
evaluates an operator of the method (no quadrature, SBP operator, PKD basis, metric term, flux).

Recipes:
  * split-Cartesian periodic meshes, 2 triangles per square / 6 Kuhn tetrahedra per cube,
    element index slab-major (x_d slowest), canonical local vertex order (reading R11);
  * warps: the BASELINE.json sine warp (R13) and the paper's sequential warp with (x - L/2)
    centring (R13);
  * initial states: density wave, Taylor-Green vortex as printed (R15),
    isentropic vortex (R14), uniform free stream;
  * perturbation for seeds >= 1.
"""
from __future__ import annotations

import itertools
import math

import numpy as np

GAMMA = 1.4


# ----------------------------------------------------------------------------------------------
# meshes
# ----------------------------------------------------------------------------------------------
def split_cartesian(d: int, M: int, L: float):
    """Periodic split-Cartesian mesh of (0,L)^d with M cells per direction.

    Returns dict(elem_vertices [ne][d+1] int64 periodic global vertex ids in canonical order,
    elem_vertex_coords [ne][d+1][d] unwrapped corner coordinates, period [d]).
    Canonical order (R11): ascending global id; if the corner simplex is negatively oriented,
    swap the first two vertices.
    """
    if M < 3:
        raise ValueError("M >= 3 required so that periodic vertex ids within an element differ")
    h = L / M
    ev, evx = [], []
    if d == 2:
        for j in range(M):
            for i in range(M):
                corners = {
                    (0, 0): (i, j), (1, 0): (i + 1, j), (1, 1): (i + 1, j + 1), (0, 1): (i, j + 1)}
                # diagonal (i,j)-(i+1,j+1) (R12)
                for tri in (((0, 0), (1, 0), (1, 1)), ((0, 0), (1, 1), (0, 1))):
                    ids, xs = [], []
                    for c in tri:
                        a, b = corners[c]
                        ids.append((a % M) + M * (b % M))
                        xs.append((a * h, b * h))
                    ev.append(ids)
                    evx.append(xs)
    elif d == 3:
        perms = list(itertools.permutations(range(3)))
        for k in range(M):
            for j in range(M):
                for i in range(M):
                    base = np.array([i, j, k])
                    for perm in perms:  # Kuhn split along the main diagonal (R12)
                        pts = [base.copy()]
                        cur = base.copy()
                        for ax in perm:
                            cur = cur.copy()
                            cur[ax] += 1
                            pts.append(cur)
                        ids = [int((p[0] % M) + M * (p[1] % M) + M * M * (p[2] % M)) for p in pts]
                        ev.append(ids)
                        evx.append([tuple(float(v) * h for v in p) for p in pts])
    else:
        raise ValueError("d must be 2 or 3")
    ev = np.array(ev, dtype=np.int64)
    evx = np.array(evx, dtype=np.float64)
    # canonical order
    order = np.argsort(ev, axis=1, kind="stable")
    ev = np.take_along_axis(ev, order, axis=1)
    evx = np.take_along_axis(evx, order[:, :, None], axis=1)
    A = evx[:, 1:, :] - evx[:, :1, :]
    det = np.linalg.det(A)
    neg = det < 0
    ev[neg, 0], ev[neg, 1] = ev[neg, 1].copy(), ev[neg, 0].copy()
    tmp = evx[neg, 0, :].copy()
    evx[neg, 0, :] = evx[neg, 1, :]
    evx[neg, 1, :] = tmp
    return dict(d=d, M=M, L=L, elem_vertices=np.ascontiguousarray(ev),
                elem_vertex_coords=np.ascontiguousarray(evx),
                period=np.full(d, float(L)))


# ----------------------------------------------------------------------------------------------
# warps (the user geometry map); all vanish on the boundary of (0,L)^d so periodic faces match
# ----------------------------------------------------------------------------------------------
def identity_map(x):
    return np.array(x, dtype=np.float64, copy=True)


def bj_warp(d: int, L: float, M: int):
    """BASELINE.json warp (R13): 2D x += 0.05 sin(pi x) sin(pi y) (and y likewise) on [0,2]^2;
    3D x_i += 0.05 h sin(x1) sin(x2) sin(x3) on [0,2pi]^3 with h = L/M.  Both factors use the
    unwarped coordinates; the 2D form is written for general L as 0.05 sin(2 pi x/L) sin(2 pi y/L)
    scaled so that L = 2 reproduces the BASELINE formula exactly."""
    def f2(x):
        x = np.asarray(x, dtype=np.float64)
        s = 0.05 * np.sin(2.0 * math.pi * x[:, 0] / L) * np.sin(2.0 * math.pi * x[:, 1] / L)
        return x + s[:, None]

    def f3(x):
        x = np.asarray(x, dtype=np.float64)
        h = L / M
        k = 2.0 * math.pi / L
        s = 0.05 * h * np.sin(k * x[:, 0]) * np.sin(k * x[:, 1]) * np.sin(k * x[:, 2])
        return x + s[:, None]
    return f2 if d == 2 else f3


def paper_warp(d: int, L: float, eps: float = 1.0 / 16.0):
    """The paper's sequential warp with (x - L/2) centring in every factor (R13)."""
    c = L / 2.0
    pi = math.pi

    def f2(x):
        x = np.asarray(x, dtype=np.float64)
        x1, x2 = x[:, 0], x[:, 1]
        t1 = x1 + eps * L * np.cos(pi / L * (x1 - c)) * np.cos(3 * pi / L * (x2 - c))
        t2 = x2 + eps * L * np.sin(4 * pi / L * (t1 - c)) * np.cos(pi / L * (x2 - c))
        return np.stack([t1, t2], axis=1)

    def f3(x):
        x = np.asarray(x, dtype=np.float64)
        x1, x2, x3 = x[:, 0], x[:, 1], x[:, 2]
        t2 = x2 + eps * L * np.cos(3 * pi / L * (x1 - c)) * np.cos(pi / L * (x2 - c)) * np.cos(pi / L * (x3 - c))
        t1 = x1 + eps * L * np.cos(pi / L * (x1 - c)) * np.sin(4 * pi / L * (t2 - c)) * np.cos(pi / L * (x3 - c))
        t3 = x3 + eps * L * np.cos(pi / L * (t1 - c)) * np.cos(2 * pi / L * (t2 - c)) * np.cos(pi / L * (x3 - c))
        return np.stack([t1, t2, t3], axis=1)
    return f2 if d == 2 else f3


# ----------------------------------------------------------------------------------------------
# initial states (conservative variables)
# ----------------------------------------------------------------------------------------------
def prim_to_cons(rho, v, p, gamma=GAMMA):
    rho = np.asarray(rho, dtype=np.float64)
    v = np.asarray(v, dtype=np.float64)
    p = np.asarray(p, dtype=np.float64)
    E = p / (gamma - 1.0) + 0.5 * rho * np.sum(v * v, axis=-1)
    return np.concatenate([rho[..., None], rho[..., None] * v, E[..., None]], axis=-1)


def density_wave(x, L=2.0):
    """rho = 1 + 0.2 sin(2 pi/L sum x), v = (1,...,1), p = 1."""
    x = np.asarray(x)
    d = x.shape[-1]
    rho = 1.0 + 0.2 * np.sin(2.0 * math.pi / L * np.sum(x, axis=-1))
    v = np.ones(x.shape[:-1] + (d,))
    return prim_to_cons(rho, v, np.ones(x.shape[:-1]))


def taylor_green(x, Ma=0.1, gamma=GAMMA):
    """P:940-941 as printed (R15)."""
    x = np.asarray(x)
    x1, x2, x3 = x[..., 0], x[..., 1], x[..., 2]
    v = np.stack([np.sin(x1) * np.cos(x2) * np.cos(x3), -np.cos(x1) * np.sin(x2) * np.cos(x3),
                  np.zeros_like(x1)], axis=-1)
    p = 1.0 / (gamma * Ma ** 2) + (np.cos(2 * x1) + 2 * np.cos(2 * x2) + np.cos(2 * x1) * np.cos(2 * x3)
                                   + np.cos(2 * x2) * np.cos(2 * x3)) / 16.0
    return prim_to_cons(np.ones_like(x1), v, p, gamma)


def kelvin_helmholtz(x, gamma=GAMMA):
    """P:931-936 (robustness test): B = tanh(15(x2 - 1/2)) - tanh(15(x2 - 3/2)),
    rho = 1/2 + 3/4 B, v = ((B - 1)/2, sin(2 pi x1)/10), p = 1 on (0, 2)^2."""
    x = np.asarray(x)
    x1, x2 = x[..., 0], x[..., 1]
    B = np.tanh(15.0 * (x2 - 0.5)) - np.tanh(15.0 * (x2 - 1.5))
    v = np.stack([0.5 * (B - 1.0), 0.1 * np.sin(2.0 * math.pi * x1)], axis=-1)
    return prim_to_cons(0.5 + 0.75 * B, v, np.ones_like(x1), gamma)


def isentropic_vortex(x, L, gamma=GAMMA, beta=1.0):
    """R14: exact translating isentropic vortex, centre (L/2, L/2), radius L/10, Mach-0.5 background."""
    x = np.asarray(x)
    R = L / 10.0
    x0 = L / 2.0
    dx, dy = (x[..., 0] - x0) / R, (x[..., 1] - x0) / R
    r2 = dx * dx + dy * dy
    T = 1.0 - (gamma - 1.0) * beta ** 2 / (8.0 * gamma * math.pi ** 2) * np.exp(1.0 - r2)
    rho = T ** (1.0 / (gamma - 1.0))
    p = rho ** gamma
    vinf = 0.5 * math.sqrt(gamma)
    a = beta / (2.0 * math.pi) * np.exp(0.5 * (1.0 - r2))
    v = np.stack([vinf - a * dy, a * dx], axis=-1)
    return prim_to_cons(rho, v, p, gamma)


def free_stream(x, d):
    x = np.asarray(x)
    v = np.zeros(x.shape[:-1] + (d,))
    v[..., 0] = 0.6
    v[..., 1] = -0.35
    if d == 3:
        v[..., 2] = 0.2
    return prim_to_cons(np.full(x.shape[:-1], 1.3), v, np.full(x.shape[:-1], 0.9))


# ----------------------------------------------------------------------------------------------
# modal-array helpers (layout contract of the ABI, not method arithmetic)
# ----------------------------------------------------------------------------------------------
def multi_index_degrees(d: int, p: int):
    """Total degree |alpha| of each modal index in the ABI's alpha1-major nested order (R9)."""
    deg = []
    for a1 in range(p + 1):
        for a2 in range(p - a1 + 1):
            if d == 2:
                deg.append(a1 + a2)
            else:
                for a3 in range(p - a1 - a2 + 1):
                    deg.append(a1 + a2 + a3)
    return np.array(deg)


def perturb_modal(u, d, p, seed, amp=1e-3):
    """Seeded perturbation for seeds >= 1: u[k,e,i] += amp |u[k,e,0]| xi/(1+deg i)^2,
    xi ~ N(0,1) drawn over the global array (partition independent)."""
    u = np.array(u, dtype=np.float64, copy=True)
    if seed == 0:
        return u
    rng = np.random.default_rng(seed)
    xi = rng.standard_normal(u.shape)
    deg = multi_index_degrees(d, p)
    scale = amp * np.abs(u[:, :, :1]) / (1.0 + deg[None, None, :]) ** 2
    scale[:, :, 0] = 0.0
    return u + scale * xi


def random_states(n, d, seed, gamma=GAMMA, spread=0.3):
    """Random admissible conservative states (for pointwise flux tests)."""
    rng = np.random.default_rng(seed)
    rho = np.exp(rng.uniform(-spread, spread, n)) * 1.1
    p = np.exp(rng.uniform(-spread, spread, n)) * 0.9
    v = rng.uniform(-0.8, 0.8, (n, d))
    return prim_to_cons(rho, v, p, gamma)


def reference_measure(d):
    """|reference simplex| = 2 (triangle) or 4/3 (tetrahedron); the constant orthonormal mode has
    the value 1/sqrt(|ref|) (layout contract of the modal arrays)."""
    return 2.0 if d == 2 else 4.0 / 3.0


def modal_state_from_centroids(mesh, p, kind, seed=0, amp=2e-2, gamma=GAMMA):
    """Synthetic modal coefficients for large meshes without evaluating any operator of the method:
    the constant mode carries the analytic state (kind = 'tgv', 'density_wave', 'vortex') at the
    element centroid (divided by the constant-mode value), higher modes are seeded Gaussian noise
    scaled amp*|mean|/(1+deg)^2.  Value distributions follow the named workload."""
    d = mesh["d"]
    L = mesh["L"]
    cen = mesh["elem_vertex_coords"].mean(axis=1)
    if kind == "tgv":
        U = taylor_green(cen, Ma=0.1, gamma=gamma)
    elif kind == "density_wave":
        U = density_wave(cen, L)
    elif kind == "vortex":
        U = isentropic_vortex(cen, L, gamma)
    else:
        U = free_stream(cen, d)
    deg = multi_index_degrees(d, p)
    ne, Nc, Np = len(cen), d + 2, len(deg)
    u = np.zeros((ne, Nc, Np))
    u[:, :, 0] = U * math.sqrt(reference_measure(d))
    rng = np.random.default_rng(seed + 1000)
    scale = amp * np.abs(u[:, :, :1]) / (1.0 + deg[None, None, :]) ** 2
    scale[:, :, 0] = 0.0
    # keep the kinetic energy perturbation small relative to pressure for admissibility
    return u + scale * rng.standard_normal(u.shape)

