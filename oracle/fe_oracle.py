"""TEST INFRASTRUCTURE ONLY — P1 finite-element restatement of the eddy-current
system used by the north-star path.

The reference ships no FE model (SPEC.md:8,13,120 put assembly out of scope);
the math restated here is PAPER.md:84-94 for a 2D A_z nodal discretisation:

    M_ij = int sigma w_i w_j,   K_ij = int nu grad w_i . grad w_j,
    r_i  = int J_s w_i,         homogeneous Dirichlet on the square boundary.

Written as a plain element loop (deliberately NOT the vectorised construction
the product uses) so the two implementations check each other.

Mesh: unit square, n x n cells, each cell split along (i,j)->(i+1,j+1).
Nodes lexicographic (x fastest): id = j*(n+1)+i.  Unknowns are the interior
nodes 1<=i,j<=n-1, numbered (j-1)*(n-1)+(i-1).  Elements: cell c=j*n+i gives
2c = (ll, lr, ur) and 2c+1 = (ll, ur, ul).

Design decisions (unspecified in BASELINE.json, recorded in DESIGN.md):
  * quad4 layout (configs 0/1): region = [cx>1/2] + 2[cy>1/2]; sigma>0 only in
    regions 0 and 3; source current in region 1.
  * blocks8 layout (configs 2/4): region = floor(4cx) + 4 floor(2cy); all
    regions conducting; source in region 1.
  * kl64 layout (config 3): sigma_e = sigma0 exp(0.3 sum_k sqrt(lam_k) xi_k
    phi_k(c_e)), phi_k separable L2-normalised cosines over (a,b) in {0..7}^2
    ordered by (a+b, a), lam_k = k^-2 / sum_j j^-2; nu = nu0; source = quad4
    region 1.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np
import scipy.sparse as sp

NU0 = 1.0 / (4.0 * math.pi * 1e-7 * 1000.0)
SIGMA0 = 1.0e6
FREQ = 50.0
PERIOD = 1.0 / FREQ
J0 = 1.0e6
KL_MODES = 64
KL_SCALE = 0.3


@dataclass
class OracleMesh:
    n: int
    xy: np.ndarray          # (n_nodes, 2)
    tri: np.ndarray         # (n_elem, 3) node ids
    centroid: np.ndarray    # (n_elem, 2)
    interior: np.ndarray    # (n_nodes,) interior index or -1

    @property
    def n_interior(self) -> int:
        return (self.n - 1) ** 2


def build_mesh(n: int) -> OracleMesh:
    if n < 2:
        raise ValueError("need at least 2 cells per side")
    n1 = n + 1
    xy = np.empty((n1 * n1, 2))
    for j in range(n1):
        for i in range(n1):
            xy[j * n1 + i] = (i / n, j / n)
    tris = []
    for j in range(n):
        for i in range(n):
            ll = j * n1 + i
            lr = ll + 1
            ul = ll + n1
            ur = ul + 1
            tris.append((ll, lr, ur))
            tris.append((ll, ur, ul))
    tri = np.array(tris, dtype=np.int64)
    cen = np.empty((len(tris), 2))
    for e, (a, b, c) in enumerate(tris):
        cen[e] = (xy[a] + xy[b] + xy[c]) / 3.0
    interior = -np.ones(n1 * n1, dtype=np.int64)
    for j in range(1, n):
        for i in range(1, n):
            interior[j * n1 + i] = (j - 1) * (n - 1) + (i - 1)
    return OracleMesh(n=n, xy=xy, tri=tri, centroid=cen, interior=interior)


def _local_matrices(p: np.ndarray):
    """P1 element mass (without sigma) and stiffness (without nu)."""
    d1 = p[1] - p[0]
    d2 = p[2] - p[0]
    jac = np.array([[d1[0], d2[0]], [d1[1], d2[1]]])
    det = np.linalg.det(jac)
    area = abs(det) / 2.0
    ref_grad = np.array([[-1.0, -1.0], [1.0, 0.0], [0.0, 1.0]])
    grads = ref_grad @ np.linalg.inv(jac)          # rows: grad lambda_a
    kloc = area * (grads @ grads.T)
    mloc = area / 12.0 * (np.ones((3, 3)) + np.eye(3))
    return mloc, kloc, area


def region_quad4(mesh: OracleMesh) -> np.ndarray:
    reg = np.empty(len(mesh.tri), dtype=np.int64)
    for e, (cx, cy) in enumerate(mesh.centroid):
        reg[e] = (1 if cx > 0.5 else 0) + (2 if cy > 0.5 else 0)
    return reg


def region_blocks8(mesh: OracleMesh) -> np.ndarray:
    reg = np.empty(len(mesh.tri), dtype=np.int64)
    for e, (cx, cy) in enumerate(mesh.centroid):
        reg[e] = min(int(4.0 * cx), 3) + 4 * min(int(2.0 * cy), 1)
    return reg


def kl_modes() -> list[tuple[int, int]]:
    pairs = [(a, b) for a in range(8) for b in range(8)]
    pairs.sort(key=lambda ab: (ab[0] + ab[1], ab[0]))
    return pairs


def kl_log_sigma(mesh: OracleMesh, xi: np.ndarray) -> np.ndarray:
    """log sigma_e for the config-3 lognormal field (per element)."""
    modes = kl_modes()
    norm = sum(1.0 / (k * k) for k in range(1, KL_MODES + 1))
    cx, cy = mesh.centroid[:, 0], mesh.centroid[:, 1]
    acc = np.zeros(len(mesh.tri))
    for k, (a, b) in enumerate(modes, start=1):
        lam = 1.0 / (k * k) / norm
        ca = 1.0 if a == 0 else math.sqrt(2.0)
        cb = 1.0 if b == 0 else math.sqrt(2.0)
        phi = ca * cb * np.cos(math.pi * a * cx) * np.cos(math.pi * b * cy)
        acc += math.sqrt(lam) * xi[k - 1] * phi
    return math.log(SIGMA0) + KL_SCALE * acc


def material_fields(mesh: OracleMesh, layout: str, params: np.ndarray):
    """Per-element (sigma_e, nu_e) from one sample's parameter vector."""
    params = np.asarray(params, dtype=float)
    if layout == "quad4":
        reg = region_quad4(mesh)
        mask = np.array([1.0, 0.0, 0.0, 1.0])
        nu = params[:4][reg]
        sigma = (params[4:8] * mask)[reg]
    elif layout == "blocks8":
        reg = region_blocks8(mesh)
        nu = params[:8][reg]
        sigma = params[8:16][reg]
    elif layout == "kl64":
        sigma = np.exp(kl_log_sigma(mesh, params))
        nu = np.full(len(mesh.tri), NU0)
    else:
        raise ValueError(f"unknown layout {layout!r}")
    return sigma, nu


def source_elements(mesh: OracleMesh, layout: str) -> np.ndarray:
    if layout in ("quad4", "kl64"):
        return region_quad4(mesh) == 1
    if layout == "blocks8":
        return region_blocks8(mesh) == 1
    raise ValueError(f"unknown layout {layout!r}")


class ElementGeometry:
    """Per-element local matrices and interior scatter lists, built once per
    mesh by an element loop; per-sample assembly only rescales them."""

    def __init__(self, mesh: OracleMesh):
        self.mesh = mesh
        rows, cols, elem, mw, kw = [], [], [], [], []
        self.src_rows, self.src_elem, self.src_w = [], [], []
        for e, nodes in enumerate(mesh.tri):
            mloc, kloc, area = _local_matrices(mesh.xy[nodes])
            gi = mesh.interior[nodes]
            for a in range(3):
                if gi[a] < 0:
                    continue
                self.src_rows.append(gi[a])
                self.src_elem.append(e)
                self.src_w.append(area / 3.0)
                for b in range(3):
                    if gi[b] < 0:
                        continue
                    rows.append(gi[a])
                    cols.append(gi[b])
                    elem.append(e)
                    mw.append(mloc[a, b])
                    kw.append(kloc[a, b])
        self.rows = np.array(rows)
        self.cols = np.array(cols)
        self.elem = np.array(elem)
        self.mw = np.array(mw)
        self.kw = np.array(kw)
        self.src_rows = np.array(self.src_rows)
        self.src_elem = np.array(self.src_elem)
        self.src_w = np.array(self.src_w)


def assemble(geom: ElementGeometry, sigma_e: np.ndarray, nu_e: np.ndarray,
             src_mask: np.ndarray, j0: float = J0):
    """Interior-reduced (M, K, profile): M/K scipy CSR, profile ndarray."""
    nint = geom.mesh.n_interior
    shape = (nint, nint)
    mass = sp.csr_matrix((sigma_e[geom.elem] * geom.mw, (geom.rows, geom.cols)), shape=shape)
    stiff = sp.csr_matrix((nu_e[geom.elem] * geom.kw, (geom.rows, geom.cols)), shape=shape)
    mass.sum_duplicates()
    stiff.sum_duplicates()
    profile = np.zeros(nint)
    for r, e, w in zip(geom.src_rows, geom.src_elem, geom.src_w):
        if src_mask[e]:
            profile[r] += j0 * w
    return mass, stiff, profile


def magnetic_energy(stiffness, a: np.ndarray) -> float:
    """W = 1/2 a^T K a (new QoI kind; no reference counterpart)."""
    return 0.5 * float(a @ (stiffness @ a))
