"""Mesh, sparsity pattern and assembly gather map of the 2D P1 eddy-current
system (host-side setup, computed once per mesh; the per-sample assembly runs
on the device in ``mlmcp_assemble``).

The reference has no FE model; the discretisation follows
PAPER.md:84-94 (M_ij = int sigma w_i w_j, K_ij = int nu grad w_i . grad w_j,
r_i = int J_s w_i) on the BASELINE.json meshes: unit square, n x n cells,
each split along (i,j)->(i+1,j+1), homogeneous Dirichlet boundary.  Nodes are
lexicographic (x fastest); unknowns are interior nodes
(j-1)(n-1)+(i-1).  Element 2c is (ll, lr, ur), 2c+1 is (ll, ur, ul) for cell
c = j*n + i.

Region layouts / material maps (design decisions):
  quad4    (configs 0/1): region = [cx>1/2] + 2[cy>1/2]; sigma>0 in regions 0, 3;
           source in region 1; params = (nu_0..nu_3, sigma_0..sigma_3).
  blocks8  (configs 2/4): region = floor(4cx) + 4 floor(2cy); all conducting;
           source in region 1; params = (nu_0..nu_7, sigma_0..sigma_7).
  kl64     (config 3): sigma_e = sigma0 exp(0.3 sum_k sqrt(lam_k) xi_k phi_k(c_e)),
           nu = nu0; source = quad4 region 1; params = xi (64 standard normals).
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

NU0 = 1.0 / (4.0 * math.pi * 1e-7 * 1000.0)
SIGMA0 = 1.0e6
FREQ = 50.0
PERIOD = 1.0 / FREQ
J0 = 1.0e6
KL_MODES = 64
KL_SCALE = 0.3

LAYOUTS = ("quad4", "blocks8", "kl64")


@dataclass
class StructuredMesh:
    """Interior-reduced P1 system structure shared by every sample."""

    n: int
    xy: np.ndarray = field(repr=False)
    tri: np.ndarray = field(repr=False)
    centroid: np.ndarray = field(repr=False)
    area: np.ndarray = field(repr=False)
    interior: np.ndarray = field(repr=False)
    row_ptr: np.ndarray = field(repr=False)
    col: np.ndarray = field(repr=False)
    # gather map: for CSR entry q, contributions cptr[q]:cptr[q+1]
    cptr: np.ndarray = field(repr=False)
    celem: np.ndarray = field(repr=False)
    cmw: np.ndarray = field(repr=False)
    ckw: np.ndarray = field(repr=False)

    @property
    def n_rows(self) -> int:
        return (self.n - 1) ** 2

    @property
    def nnz(self) -> int:
        return int(self.row_ptr[-1])

    @property
    def n_elem(self) -> int:
        return len(self.tri)


def structured_mesh(n: int) -> StructuredMesh:
    if n < 2:
        raise ValueError(f"need n >= 2 cells per side, got {n}")
    n1 = n + 1
    jj, ii = np.meshgrid(np.arange(n1), np.arange(n1), indexing="ij")
    xy = np.stack([ii.ravel() / n, jj.ravel() / n], axis=1)
    cj, ci = np.meshgrid(np.arange(n), np.arange(n), indexing="ij")
    ll = (cj * n1 + ci).ravel()
    lr, ul = ll + 1, ll + n1
    ur = ul + 1
    tri = np.empty((2 * n * n, 3), dtype=np.int64)
    tri[0::2] = np.stack([ll, lr, ur], axis=1)
    tri[1::2] = np.stack([ll, ur, ul], axis=1)
    p = xy[tri]                                   # (E, 3, 2)
    centroid = (p[:, 0] + p[:, 1] + p[:, 2]) / 3.0
    d1 = p[:, 1] - p[:, 0]
    d2 = p[:, 2] - p[:, 0]
    det = d1[:, 0] * d2[:, 1] - d1[:, 1] * d2[:, 0]
    area = np.abs(det) / 2.0
    g1 = np.stack([d2[:, 1], -d2[:, 0]], axis=1) / det[:, None]
    g2 = np.stack([-d1[:, 1], d1[:, 0]], axis=1) / det[:, None]
    grads = np.stack([-(g1 + g2), g1, g2], axis=1)          # (E, 3, 2)
    kloc = area[:, None, None] * np.einsum("eak,ebk->eab", grads, grads)
    mloc = (area / 12.0)[:, None, None] * (np.ones((3, 3)) + np.eye(3))[None]

    interior = -np.ones(n1 * n1, dtype=np.int64)
    inner = (jj[1:n, 1:n] * n1 + ii[1:n, 1:n]).ravel()
    interior[inner] = np.arange(len(inner))
    gi = interior[tri]                                       # (E, 3)
    e_idx, a_idx, b_idx = np.nonzero((gi[:, :, None] >= 0) & (gi[:, None, :] >= 0))
    rows = gi[e_idx, a_idx]
    cols = gi[e_idx, b_idx]
    nrow = (n - 1) ** 2
    key = rows * nrow + cols
    uniq, inv = np.unique(key, return_inverse=True)
    row_of = uniq // nrow
    col_of = uniq % nrow
    row_ptr = np.zeros(nrow + 1, dtype=np.int64)
    np.add.at(row_ptr, row_of + 1, 1)
    row_ptr = np.cumsum(row_ptr)
    order = np.lexsort((e_idx, inv))                         # by CSR entry, then element
    q_sorted = inv[order]
    cptr = np.zeros(len(uniq) + 1, dtype=np.int64)
    np.add.at(cptr, q_sorted + 1, 1)
    cptr = np.cumsum(cptr)
    return StructuredMesh(
        n=n, xy=xy, tri=tri, centroid=centroid, area=area, interior=interior,
        row_ptr=row_ptr.astype(np.int32), col=col_of.astype(np.int32),
        cptr=cptr.astype(np.int32), celem=e_idx[order].astype(np.int32),
        cmw=mloc[e_idx, a_idx, b_idx][order], ckw=kloc[e_idx, a_idx, b_idx][order])


def region_map(mesh: StructuredMesh, layout: str) -> np.ndarray:
    cx, cy = mesh.centroid[:, 0], mesh.centroid[:, 1]
    if layout in ("quad4", "kl64"):
        return ((cx > 0.5).astype(np.int32) + 2 * (cy > 0.5).astype(np.int32)).astype(np.int32)
    if layout == "blocks8":
        return (np.minimum((4.0 * cx).astype(np.int32), 3)
                + 4 * np.minimum((2.0 * cy).astype(np.int32), 1)).astype(np.int32)
    raise ValueError(f"unknown layout {layout!r}")


def conducting_mask(layout: str) -> np.ndarray:
    if layout == "quad4":
        return np.array([1.0, 0.0, 0.0, 1.0])
    if layout == "blocks8":
        return np.ones(8)
    raise ValueError(f"layout {layout!r} has no region conductivity mask")


def n_params(layout: str) -> int:
    return {"quad4": 8, "blocks8": 16, "kl64": KL_MODES}[layout]


def source_profile(mesh: StructuredMesh, layout: str, j0: float = J0) -> np.ndarray:
    """r(t) = sin(2 pi f t) * profile with profile_i = sum_{e in src, i in e} J0 |e|/3."""
    src = region_map(mesh, "quad4" if layout == "kl64" else layout) == 1
    gi = mesh.interior[mesh.tri]
    prof = np.zeros(mesh.n_rows)
    w = np.repeat((j0 * mesh.area / 3.0)[:, None], 3, axis=1)
    sel = src[:, None] & (gi >= 0)
    np.add.at(prof, gi[sel], w[sel])
    return prof


# element slots of the region-linear operator of one interior point (i, j):
# the six triangles around the node in increasing element index —
# lower/upper of cell (i-1, j-1), upper of (i, j-1), lower of (i-1, j),
# lower/upper of (i, j) — and the subsets each stencil coefficient sums over
# (the hypotenuse entry NE couples the two triangles of the node's own cell)
REGION_SLOTS = {"C": (0, 1, 2, 3, 4, 5), "E": (2, 4), "N": (3, 5), "NE": (4, 5)}


@dataclass
class RegionGrid:
    """Region-linear description of the per-sample operator on a structured
    grid: coefficient c of point p is  sum_e sigma_{r(e)} mw[c][e]  (mass) and
    sum_e nu_{r(e)} kw[c][e]  (stiffness) over the slot's triangles, summed in
    the assembly gather map's element order (bitwise the CSR values when
    ``bitwise``).  code[p] packs the six triangles' regions, 4 bits each."""

    code: np.ndarray        # uint32 [n_rows]
    mw: np.ndarray          # [12]: C0..C5, E0, E1, N0, N1, NE0, NE1
    kw: np.ndarray          # [12]
    n_regions: int
    bitwise: bool


def region_grid(mesh: StructuredMesh, region: np.ndarray, n_regions: int):
    """RegionGrid of a region-constant material layout, or None when the gather
    map does not have the structured-grid form (checked entry by entry)."""
    n, w = mesh.n, mesh.n - 1
    if n_regions > 16 or w < 2:
        return None
    N = mesh.n_rows
    p = np.arange(N)
    i, j = p % w + 1, p // w + 1
    csw, cs, cw, co = (j - 1) * n + i - 1, (j - 1) * n + i, j * n + i - 1, j * n + i
    E6 = np.stack([2 * csw, 2 * csw + 1, 2 * cs + 1, 2 * cw, 2 * co, 2 * co + 1], axis=1)
    rp, col, cptr = mesh.row_ptr.astype(np.int64), mesh.col, mesh.cptr.astype(np.int64)
    mw, kw = np.zeros(12), np.zeros(12)
    bitwise = True
    base = 0
    for name, off, es in (("C", 0, REGION_SLOTS["C"]), ("E", 1, REGION_SLOTS["E"]),
                          ("N", w, REGION_SLOTS["N"]), ("NE", w + 1, REGION_SLOTS["NE"])):
        has = np.ones(N, dtype=bool)
        if name in ("E", "NE"):
            has &= i + 1 < n
        if name in ("N", "NE"):
            has &= j + 1 < n
        pp = p[has]
        # CSR position of (pp, pp + off): columns are sorted per row
        q = np.full(len(pp), -1, dtype=np.int64)
        for d in range(int(np.max(rp[1:] - rp[:-1]))):
            cand = rp[pp] + d
            hit = (cand < rp[pp + 1]) & (col[np.minimum(cand, len(col) - 1)] == pp + off)
            q[hit] = cand[hit]
        if np.any(q < 0) or np.any(cptr[q + 1] - cptr[q] != len(es)):
            return None
        cols = np.stack([cptr[q] + t for t in range(len(es))], axis=1)
        if not np.array_equal(mesh.celem[cols], E6[pp][:, list(es)]):
            return None
        cm, ck = mesh.cmw[cols], mesh.ckw[cols]
        m0, k0 = cm[0], ck[0]
        if not (np.array_equal(cm, np.broadcast_to(m0, cm.shape))
                and np.array_equal(ck, np.broadcast_to(k0, ck.shape))):
            bitwise = False
            scale = max(np.max(np.abs(cm)), 1e-300), max(np.max(np.abs(ck)), 1e-300)
            if (np.max(np.abs(cm - m0)) > 1e-14 * scale[0]
                    or np.max(np.abs(ck - k0)) > 1e-14 * scale[1]):
                return None
        mw[base:base + len(es)] = m0
        kw[base:base + len(es)] = k0
        base += len(es)
    reg = np.asarray(region, dtype=np.int64)[E6]            # [N, 6]
    if reg.min() < 0 or reg.max() >= n_regions:
        return None
    code = np.zeros(N, dtype=np.uint64)
    for e in range(6):
        code |= reg[:, e].astype(np.uint64) << np.uint64(4 * e)
    return RegionGrid(code.astype(np.uint32), mw, kw, int(n_regions), bitwise)


def kl_basis(mesh: StructuredMesh) -> np.ndarray:
    """(KL_MODES, E): sqrt(lam_k) phi_k(c_e); modes (a,b) in {0..7}^2 ordered by
    (a+b, a); lam_k = k^-2 / sum_j j^-2; phi separable L2-normalised cosines."""
    pairs = sorted(((a, b) for a in range(8) for b in range(8)), key=lambda ab: (ab[0] + ab[1], ab[0]))
    k = np.arange(1, KL_MODES + 1, dtype=float)
    lam = (1.0 / k ** 2) / np.sum(1.0 / k ** 2)
    cx, cy = mesh.centroid[:, 0], mesh.centroid[:, 1]
    out = np.empty((KL_MODES, mesh.n_elem))
    for idx, (a, b) in enumerate(pairs):
        ca = 1.0 if a == 0 else math.sqrt(2.0)
        cb = 1.0 if b == 0 else math.sqrt(2.0)
        out[idx] = math.sqrt(lam[idx]) * ca * cb * np.cos(math.pi * a * cx) * np.cos(math.pi * b * cy)
    return out
