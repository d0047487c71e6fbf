"""Seeded synthetic inputs shared by the oracle tests, the CUDA parity tests and bench.py.

This module holds NO arithmetic of the method (no intersection, reflection,
capture, dedupe or refinement).  It only builds input clouds shaped like the
paper's indoor scenes (§IV-A, noise P:500, estimated normals
P:361) following the recipe in DESIGN.md §"Input recipe" / SURVEY.md §8(d):

  C1  analytic box room 4x3x2.5 m, 20,008 noise-free surfels, labels 0..5
  SR  synthetic room 8x6x3 m + pillar + cabinet + table, uniform random
      surfels per face (area-proportional), Gaussian noise along the true
      normal (sigma), optional PCA re-estimated normals, 20 exterior edges.

Everything is float32 / int32 numpy, seeded from SEED = 240306648.
"""
from __future__ import annotations

import dataclasses
import math

import numpy as np

SEED = 240306648


@dataclasses.dataclass
class Edges:
    """Exterior diffraction edges (§II-A, n_exp in (1,2))."""
    a: np.ndarray       # (E,3) f32 start
    b: np.ndarray       # (E,3) f32 end
    t0: np.ndarray      # (E,3) f32 face-0 tangent (perp to e, pointing into face 0)
    n0: np.ndarray      # (E,3) f32 face-0 outward normal
    n1: np.ndarray      # (E,3) f32 face-1 outward normal
    n_exp: np.ndarray   # (E,)  f32 exterior angle / pi
    label: np.ndarray   # (E,)  i32 unique edge label

    def __len__(self):
        return int(self.a.shape[0])

    @staticmethod
    def empty() -> "Edges":
        z3 = np.zeros((0, 3), np.float32)
        return Edges(z3, z3, z3, z3, z3, np.zeros(0, np.float32), np.zeros(0, np.int32))


@dataclasses.dataclass
class Scene:
    points: np.ndarray   # (N,3) f32
    normals: np.ndarray  # (N,3) f32
    radii: np.ndarray    # (N,)  f32
    labels: np.ndarray   # (N,)  i32
    edges: Edges
    name: str = ""

    @property
    def n(self) -> int:
        return int(self.points.shape[0])


@dataclasses.dataclass
class LaunchCase:
    """One workload: a scene plus the launch / refine parameters."""
    name: str
    scene: Scene
    tx: np.ndarray            # (3,) f32
    rx: np.ndarray            # (R,3) f32
    n_rays: int
    max_refl: int
    max_diff: int
    voxel: float
    kappa: int = 1
    tau: float = 0.0015
    c_R: float = 1.0
    dphi_deg: float = 2.5
    theta_ex_deg: float = 25.0
    edge_bin: float = 0.25
    # refinement (Table I/II P:373)
    xi: float = 2.0
    r_s: float = 0.003
    sigma_noise: float = 0.0


# --------------------------------------------------------------------------
# planar rectangle sampling helpers (pure geometry of the synthetic inputs)
# --------------------------------------------------------------------------

def _rect_grid(c, U, V, nu, nv):
    """Cell-centred regular grid on the rectangle c + a*U + b*V, a,b in [0,1]."""
    a = (np.arange(nu, dtype=np.float64) + 0.5) / nu
    b = (np.arange(nv, dtype=np.float64) + 0.5) / nv
    A, B = np.meshgrid(a, b, indexing="ij")
    return (np.asarray(c, np.float64)[None, :] + A.reshape(-1, 1) * np.asarray(U, np.float64)[None, :]
            + B.reshape(-1, 1) * np.asarray(V, np.float64)[None, :])


def box_room(density: int = 1) -> Scene:
    """C1: box [0,4]x[0,3]x[0,2.5] m, inward normals, regular cell-centred grids.

    floor/ceiling 74x55, x-walls 55x46, y-walls 74x46 -> 20,008 surfels, r = 0.042 m,
    labels 0..5 (x=0, x=4, y=0, y=3, z=0, z=2.5).  density k multiplies the grid counts per
    axis by k (and divides r by k): the dense variants the point-set SDF intersection (NEXT-1)
    needs — its AABB primitives must hold several points each."""
    X, Y, Z = 4.0, 3.0, 2.5
    faces = [
        # (corner, U, V, nu, nv, normal, label)
        ((0, 0, 0), (0, Y, 0), (0, 0, Z), 55, 46, (1, 0, 0), 0),
        ((X, 0, 0), (0, Y, 0), (0, 0, Z), 55, 46, (-1, 0, 0), 1),
        ((0, 0, 0), (X, 0, 0), (0, 0, Z), 74, 46, (0, 1, 0), 2),
        ((0, Y, 0), (X, 0, 0), (0, 0, Z), 74, 46, (0, -1, 0), 3),
        ((0, 0, 0), (X, 0, 0), (0, Y, 0), 74, 55, (0, 0, 1), 4),
        ((0, 0, Z), (X, 0, 0), (0, Y, 0), 74, 55, (0, 0, -1), 5),
    ]
    P, N, L = [], [], []
    for c, U, V, nu, nv, nrm, lab in faces:
        p = _rect_grid(c, U, V, nu * density, nv * density)
        P.append(p)
        N.append(np.repeat(np.asarray(nrm, np.float64)[None, :], p.shape[0], 0))
        L.append(np.full(p.shape[0], lab, np.int32))
    P = np.concatenate(P).astype(np.float32)
    N = np.concatenate(N).astype(np.float32)
    L = np.concatenate(L)
    R = np.full(P.shape[0], 0.042 / density, np.float32)
    return Scene(P, N, R, L, Edges.empty(), "box_room" if density == 1 else f"box_room(x{density})")


# --------------------------------------------------------------------------
# synthetic room (SR)
# --------------------------------------------------------------------------

_ROOM = (8.0, 6.0, 3.0)
_PILLAR = ((3.6, 2.6, 0.0), (4.2, 3.2, 3.0))
_CABINET = ((6.0, 0.8, 0.0), (7.0, 1.3, 2.0))
_TABLE = ((1.2, 3.8, 0.0), (2.8, 4.6, 0.75))


def _box_faces(lo, hi, label0, top=True, inward=False):
    """Axis-aligned box side faces (+top).  Returns list of (c,U,V,normal,label,holes)."""
    x0, y0, z0 = lo
    x1, y1, z1 = hi
    s = -1.0 if inward else 1.0
    f = [
        ((x0, y0, z0), (0, y1 - y0, 0), (0, 0, z1 - z0), (-s, 0, 0)),
        ((x1, y0, z0), (0, y1 - y0, 0), (0, 0, z1 - z0), (s, 0, 0)),
        ((x0, y0, z0), (x1 - x0, 0, 0), (0, 0, z1 - z0), (0, -s, 0)),
        ((x0, y1, z0), (x1 - x0, 0, 0), (0, 0, z1 - z0), (0, s, 0)),
    ]
    if top:
        f.append(((x0, y0, z1), (x1 - x0, 0, 0), (0, y1 - y0, 0), (0, 0, s)))
    return [(c, U, V, n, label0 + k, []) for k, (c, U, V, n) in enumerate(f)]


def _sr_faces():
    X, Y, Z = _ROOM
    fp_floor = [(_PILLAR[0][:2], _PILLAR[1][:2]), (_CABINET[0][:2], _CABINET[1][:2]),
                (_TABLE[0][:2], _TABLE[1][:2])]
    fp_ceil = [(_PILLAR[0][:2], _PILLAR[1][:2])]
    faces = [
        ((0, 0, 0), (0, Y, 0), (0, 0, Z), (1, 0, 0), 0, []),
        ((X, 0, 0), (0, Y, 0), (0, 0, Z), (-1, 0, 0), 1, []),
        ((0, 0, 0), (X, 0, 0), (0, 0, Z), (0, 1, 0), 2, []),
        ((0, Y, 0), (X, 0, 0), (0, 0, Z), (0, -1, 0), 3, []),
        ((0, 0, 0), (X, 0, 0), (0, Y, 0), (0, 0, 1), 4, fp_floor),
        ((0, 0, Z), (X, 0, 0), (0, Y, 0), (0, 0, -1), 5, fp_ceil),
    ]
    faces += _box_faces(_PILLAR[0], _PILLAR[1], 6, top=False)      # labels 6..9
    faces += _box_faces(_CABINET[0], _CABINET[1], 10, top=True)    # labels 10..14
    faces += _box_faces(_TABLE[0], _TABLE[1], 15, top=True)        # labels 15..19
    return faces


def _face_area(f):
    c, U, V, n, lab, holes = f
    a = float(np.linalg.norm(np.cross(U, V)))
    for (lo, hi) in holes:
        a -= (hi[0] - lo[0]) * (hi[1] - lo[1])
    return a


def _sample_face(rng, f, count):
    c, U, V, n, lab, holes = f
    out = np.zeros((0, 3))
    c = np.asarray(c, np.float64)
    U = np.asarray(U, np.float64)
    V = np.asarray(V, np.float64)
    while out.shape[0] < count:
        m = int((count - out.shape[0]) * 1.3) + 16
        ab = rng.random((m, 2))
        p = c[None] + ab[:, :1] * U[None] + ab[:, 1:] * V[None]
        keep = np.ones(m, bool)
        for (lo, hi) in holes:
            inside = (p[:, 0] > lo[0]) & (p[:, 0] < hi[0]) & (p[:, 1] > lo[1]) & (p[:, 1] < hi[1])
            keep &= ~inside
        out = np.concatenate([out, p[keep]])
    return out[:count]


def _split_counts(n, areas):
    areas = np.asarray(areas, np.float64)
    exact = n * areas / areas.sum()
    cnt = np.floor(exact).astype(np.int64)
    rem = n - cnt.sum()
    order = np.argsort(-(exact - cnt), kind="stable")
    cnt[order[:rem]] += 1
    return cnt


def sr_edges() -> Edges:
    """20 exterior (convex, n = 1.5) edges of the SR objects: 4 pillar verticals,
    4 verticals + 4 top edges for cabinet and table (DESIGN.md input recipe)."""
    A, B, T0, N0, N1, LAB = [], [], [], [], [], []

    def vert_edges(lo, hi):
        x0, y0, z0 = lo
        x1, y1, z1 = hi
        # corner (x,y), face-0 normal, face-0 tangent (into face 0 away from edge), face-1 normal
        return [
            ((x0, y0), (-1, 0, 0), (0, 1, 0), (0, -1, 0)),
            ((x1, y0), (0, -1, 0), (-1, 0, 0), (1, 0, 0)),
            ((x1, y1), (1, 0, 0), (0, -1, 0), (0, 1, 0)),
            ((x0, y1), (0, 1, 0), (1, 0, 0), (-1, 0, 0)),
        ], z0, z1

    def top_edges(lo, hi):
        x0, y0, z0 = lo
        x1, y1, z1 = hi
        # face 0 = top (normal +z), tangent into the top face; face 1 = side
        return [
            ((x0, y0, z1), (x1, y0, z1), (0, 1, 0), (0, -1, 0)),
            ((x1, y0, z1), (x1, y1, z1), (-1, 0, 0), (1, 0, 0)),
            ((x1, y1, z1), (x0, y1, z1), (0, -1, 0), (0, 1, 0)),
            ((x0, y1, z1), (x0, y0, z1), (1, 0, 0), (-1, 0, 0)),
        ]

    for lo, hi, top in ((_PILLAR[0], _PILLAR[1], False), (_CABINET[0], _CABINET[1], True),
                        (_TABLE[0], _TABLE[1], True)):
        ve, z0, z1 = vert_edges(lo, hi)
        for (xy, n0, t0, n1) in ve:
            A.append((xy[0], xy[1], z0))
            B.append((xy[0], xy[1], z1))
            N0.append(n0)
            T0.append(t0)
            N1.append(n1)
        if top:
            for (a, b, t0, n1) in top_edges(lo, hi):
                A.append(a)
                B.append(b)
                N0.append((0, 0, 1))
                T0.append(t0)
                N1.append(n1)
    E = len(A)
    LAB = 100 + np.arange(E, dtype=np.int32)
    f = lambda x: np.asarray(x, np.float32).reshape(E, 3)
    return Edges(f(A), f(B), f(T0), f(N0), f(N1), np.full(E, 1.5, np.float32), LAB)


def add_normal_noise(points, normals, sigma, seed):
    """Gaussian displacement along the (true) normal.  sigma = 0 returns
    a bit-identical cloud."""
    rng = np.random.default_rng(seed)
    g = rng.standard_normal(points.shape[0])
    p = points.astype(np.float64) + (sigma * g)[:, None] * normals.astype(np.float64)
    return p.astype(np.float32)


def pca_normals(points, ref_normals, k=16):
    """Normals re-estimated by PCA over the k nearest neighbours (harness only, PAPER.md
    P:361 used a 10 cm radius least-squares plane), flipped into ref_normals' hemisphere."""
    from scipy.spatial import cKDTree
    P = points.astype(np.float64)
    tree = cKDTree(P)
    out = np.empty_like(P)
    B = 1 << 18
    for s in range(0, P.shape[0], B):
        _, idx = tree.query(P[s:s + B], k=k, workers=-1)
        Q = P[idx]                                  # (b,k,3)
        Q = Q - Q.mean(axis=1, keepdims=True)
        C = np.einsum("bki,bkj->bij", Q, Q)
        w, v = np.linalg.eigh(C)
        nrm = v[:, :, 0]
        sgn = np.sign(np.einsum("bi,bi->b", nrm, ref_normals[s:s + B].astype(np.float64)))
        sgn[sgn == 0] = 1.0
        out[s:s + B] = nrm * sgn[:, None]
    out /= np.linalg.norm(out, axis=1, keepdims=True)
    return out.astype(np.float32)


def synth_room(n=1_000_000, sigma=0.0, seed=SEED, normals="true", k_pca=16) -> Scene:
    """SR (configs C2/C3): uniform random surfels per face with area-proportional counts,
    r = sqrt(12/(pi*rho)), one label per planar face, noise sigma (m) along true normals."""
    rng = np.random.default_rng(seed)
    faces = _sr_faces()
    areas = [_face_area(f) for f in faces]
    cnt = _split_counts(n, areas)
    P, N, L = [], [], []
    for f, c in zip(faces, cnt):
        p = _sample_face(rng, f, int(c))
        P.append(p)
        N.append(np.repeat(np.asarray(f[3], np.float64)[None], p.shape[0], 0))
        L.append(np.full(p.shape[0], f[4], np.int32))
    P = np.concatenate(P).astype(np.float32)
    Nt = np.concatenate(N).astype(np.float32)
    L = np.concatenate(L)
    rho = n / float(np.sum(areas))
    r = math.sqrt(12.0 / (math.pi * rho))
    P = add_normal_noise(P, Nt, sigma, seed + 1)
    if normals == "pca":
        Nn = pca_normals(P, Nt, k_pca)
    else:
        Nn = Nt
    R = np.full(P.shape[0], r, np.float32)
    return Scene(P, Nn, R, L, sr_edges(), f"synth_room(n={n},sigma={sigma},normals={normals})")


# --------------------------------------------------------------------------
# reconstructed-room-like RR (configs C4/C5)
# --------------------------------------------------------------------------

_DOOR = (2.5, 3.5, 2.0)  # door recess in wall x = 8: y in [2.5, 3.5], z in [0, 2], depth 0.1


def _rr_layout(seed):
    """Faces of the RR room: SR + 6 clutter boxes + a door recess, 3 wall holes, walls split
    into 2-3 labels; per-face density factor U[0.5, 2].  Returns (faces, factors, edges)."""
    rng = np.random.default_rng(seed + 7)
    X, Y, Z = _ROOM
    faces = []
    lab = 0
    # room walls (split into 2-3 labels along their horizontal axis) with holes
    walls = [((0, 0, 0), (0, Y, 0), (0, 0, Z), (1, 0, 0)), ((X, 0, 0), (0, Y, 0), (0, 0, Z), (-1, 0, 0)),
             ((0, 0, 0), (X, 0, 0), (0, 0, Z), (0, 1, 0)), ((0, Y, 0), (X, 0, 0), (0, 0, Z), (0, -1, 0))]
    hole_walls = rng.choice([0, 2, 3], 3, replace=True)
    wall_holes = {0: [], 1: [], 2: [], 3: []}
    for w in hole_walls:
        wdt, hgt = rng.uniform(0.3, 1.0, 2)
        u0 = rng.uniform(0.3, (Y if w < 2 else X) - 0.3 - wdt)
        v0 = rng.uniform(0.3, Z - 0.3 - hgt)
        wall_holes[int(w)].append(((u0, v0), (u0 + wdt, v0 + hgt)))
    wall_holes[1].append(((_DOOR[0], 0.0), (_DOOR[1], _DOOR[2])))  # the door opening
    for wi, (c, U, V, n) in enumerate(walls):
        L = float(np.linalg.norm(U))
        k = int(rng.integers(2, 4))
        cuts = np.sort(rng.uniform(0.2, 0.8, k - 1)) * L
        edges_u = np.concatenate([[0.0], cuts, [L]])
        ud = np.asarray(U, float) / L
        for s0, s1 in zip(edges_u[:-1], edges_u[1:]):
            cc = tuple(np.asarray(c, float) + s0 * ud)
            UU = tuple((s1 - s0) * ud)
            holes = [((max(h0[0], s0) - s0, h0[1]), (min(h1[0], s1) - s0, h1[1]))
                     for (h0, h1) in wall_holes[wi] if h1[0] > s0 and h0[0] < s1]
            faces.append((cc, UU, V, n, lab, holes))
            lab += 1
    # floor / ceiling with object footprints removed
    clutter = []
    for _ in range(6):
        sx, sy, sz = rng.uniform(0.2, 0.5, 3)
        if rng.random() < 0.35:  # on the table
            x0 = rng.uniform(_TABLE[0][0] + 0.05, _TABLE[1][0] - sx - 0.05)
            y0 = rng.uniform(_TABLE[0][1] + 0.02, max(_TABLE[0][1] + 0.021, _TABLE[1][1] - sy - 0.02))
            z0 = _TABLE[1][2]
        else:
            for _t in range(100):
                x0 = rng.uniform(0.3, X - 0.3 - sx)
                y0 = rng.uniform(0.3, Y - 0.3 - sy)
                boxes = [_PILLAR, _CABINET, _TABLE] + [(c_[0], c_[1]) for c_ in clutter]
                if all(x0 + sx < b[0][0] - 0.1 or x0 > b[1][0] + 0.1 or y0 + sy < b[0][1] - 0.1
                       or y0 > b[1][1] + 0.1 for b in boxes):
                    break
            z0 = 0.0
        clutter.append(((x0, y0, z0), (x0 + sx, y0 + sy, z0 + sz)))
    fp_floor = [(_PILLAR[0][:2], _PILLAR[1][:2]), (_CABINET[0][:2], _CABINET[1][:2]),
                (_TABLE[0][:2], _TABLE[1][:2])] + [(c_[0][:2], c_[1][:2]) for c_ in clutter if c_[0][2] == 0.0]
    faces.append(((0, 0, 0), (X, 0, 0), (0, Y, 0), (0, 0, 1), lab, fp_floor))
    lab += 1
    faces.append(((0, 0, Z), (X, 0, 0), (0, Y, 0), (0, 0, -1), lab, [(_PILLAR[0][:2], _PILLAR[1][:2])]))
    lab += 1
    # door recess (back, two jambs, head)
    faces.append(((X + 0.1, _DOOR[0], 0), (0, _DOOR[1] - _DOOR[0], 0), (0, 0, _DOOR[2]), (-1, 0, 0), lab, []))
    faces.append(((X, _DOOR[0], 0), (0.1, 0, 0), (0, 0, _DOOR[2]), (0, 1, 0), lab + 1, []))
    faces.append(((X, _DOOR[1], 0), (0.1, 0, 0), (0, 0, _DOOR[2]), (0, -1, 0), lab + 2, []))
    faces.append(((X, _DOOR[0], _DOOR[2]), (0.1, 0, 0), (0, _DOOR[1] - _DOOR[0], 0), (0, 0, -1), lab + 3, []))
    lab += 4
    # objects
    faces += _box_faces(_PILLAR[0], _PILLAR[1], lab, top=False)
    lab += 4
    faces += _box_faces(_CABINET[0], _CABINET[1], lab, top=True)
    lab += 5
    tb = _box_faces(_TABLE[0], _TABLE[1], lab, top=True)
    # clutter on the table: remove its footprint from the table top
    tb[-1] = tb[-1][:5] + ([(c_[0][:2], c_[1][:2]) for c_ in clutter if c_[0][2] > 0.0],)
    faces += tb
    lab += 5
    for (lo, hi) in clutter:
        faces += _box_faces(lo, hi, lab, top=True)
        lab += 5
    factors = rng.uniform(0.5, 2.0, len(faces))
    # edges: SR's 20 + clutter verticals / tops at least 0.3 m long
    E = sr_edges()
    A, B, T0, N0, N1 = [list(x) for x in (E.a, E.b, E.t0, E.n0, E.n1)]
    for (lo, hi) in clutter:
        x0, y0, z0 = lo
        x1, y1, z1 = hi
        if z1 - z0 >= 0.3:
            for (xy, n0, t0, n1) in [((x0, y0), (-1, 0, 0), (0, 1, 0), (0, -1, 0)),
                                     ((x1, y0), (0, -1, 0), (-1, 0, 0), (1, 0, 0)),
                                     ((x1, y1), (1, 0, 0), (0, -1, 0), (0, 1, 0)),
                                     ((x0, y1), (0, 1, 0), (1, 0, 0), (-1, 0, 0))]:
                A.append((xy[0], xy[1], z0)); B.append((xy[0], xy[1], z1))
                N0.append(n0); T0.append(t0); N1.append(n1)
        for (a, b, t0, n1) in [((x0, y0, z1), (x1, y0, z1), (0, 1, 0), (0, -1, 0)),
                               ((x1, y0, z1), (x1, y1, z1), (-1, 0, 0), (1, 0, 0)),
                               ((x1, y1, z1), (x0, y1, z1), (0, -1, 0), (0, 1, 0)),
                               ((x0, y1, z1), (x0, y0, z1), (1, 0, 0), (-1, 0, 0))]:
            if np.linalg.norm(np.subtract(b, a)) >= 0.3:
                A.append(a); B.append(b); N0.append((0, 0, 1)); T0.append(t0); N1.append(n1)
    ne = len(A)
    f = lambda x: np.asarray(x, np.float32).reshape(ne, 3)
    edges = Edges(f(A), f(B), f(T0), f(N0), f(N1), np.full(ne, 1.5, np.float32),
                  (1000 + np.arange(ne)).astype(np.int32))
    return faces, factors, edges, clutter


def plane_fit_normals(points, ref_normals, cell=0.10):
    """Harness normal estimation for large clouds: least-squares plane (PCA) of the points in
    each 10 cm cell (the paper's 10 cm neighbourhood), flipped into ref_normals'
    hemisphere; cells with < 3 points keep the reference normal."""
    P = points.astype(np.float64)
    key = np.floor((P - P.min(0)) / cell).astype(np.int64)
    dims = key.max(0) + 1
    lin = key[:, 0] + dims[0] * (key[:, 1] + dims[1] * key[:, 2])
    uniq, inv, cnt = np.unique(lin, return_inverse=True, return_counts=True)
    m = len(uniq)
    S = np.zeros((m, 3))
    for a in range(3):
        S[:, a] = np.bincount(inv, P[:, a], m)
    mean = S / cnt[:, None]
    C = np.zeros((m, 3, 3))
    D = P - mean[inv]
    for a in range(3):
        for b in range(a, 3):
            v = np.bincount(inv, D[:, a] * D[:, b], m)
            C[:, a, b] = v
            C[:, b, a] = v
    w, vec = np.linalg.eigh(C)
    nrm = vec[:, :, 0][inv]
    sgn = np.sign(np.einsum("ij,ij->i", nrm, ref_normals.astype(np.float64)))
    sgn[sgn == 0] = 1
    nrm *= sgn[:, None]
    bad = cnt[inv] < 3
    nrm[bad] = ref_normals[bad]
    nrm /= np.linalg.norm(nrm, axis=1, keepdims=True)
    return nrm.astype(np.float32)


def recon_room(n=10_000_000, sigma=0.010, seed=SEED, normals="fit") -> Scene:
    """RR (C4/C5): reconstructed-room-like cloud — SR + clutter + door recess, wall holes,
    walls split into 2-3 labels, per-face density U[0.5,2], per-point radius
    sqrt(12/(pi rho_face)), 0.5 % outliers (+-5 cm, random normals), Gaussian noise sigma along
    the true normal, normals re-estimated by 10 cm plane fits (true normals if normals='true')."""
    faces, factors, edges, _ = _rr_layout(seed)
    rng = np.random.default_rng(seed + 11)
    areas = np.array([_face_area(f) for f in faces])
    cnt = _split_counts(n, areas * factors)
    P, N, L, R = [], [], [], []
    for f, c, a in zip(faces, cnt, areas):
        p = _sample_face(rng, f, int(c))
        P.append(p)
        N.append(np.repeat(np.asarray(f[3], np.float64)[None], p.shape[0], 0))
        L.append(np.full(p.shape[0], f[4], np.int32))
        rho = max(1.0, c / max(a, 1e-9))
        R.append(np.full(p.shape[0], math.sqrt(12.0 / (math.pi * rho)), np.float32))
    P = np.concatenate(P)
    Nt = np.concatenate(N)
    L = np.concatenate(L)
    R = np.concatenate(R)
    P = add_normal_noise(P.astype(np.float32), Nt.astype(np.float32), sigma, seed + 1).astype(np.float64)
    n_out = int(0.005 * P.shape[0])
    idx = rng.choice(P.shape[0], n_out, replace=False)
    P[idx] += rng.uniform(-0.05, 0.05, (n_out, 3))
    P = P.astype(np.float32)
    Nn = plane_fit_normals(P, Nt) if normals == "fit" else Nt.astype(np.float32)
    rn = rng.standard_normal((n_out, 3))
    Nn[idx] = (rn / np.linalg.norm(rn, axis=1, keepdims=True)).astype(np.float32)
    return Scene(P, Nn.astype(np.float32), R.astype(np.float32), L, edges,
                 f"recon_room(n={P.shape[0]},sigma={sigma})")


def _drop_rx(rx, scene, clearance=0.3):
    """RX within `clearance` of (or inside) an object box are dropped."""
    _, _, _, clutter = _rr_layout(SEED)
    boxes = [_PILLAR, _CABINET, _TABLE] + clutter
    keep = np.ones(len(rx), bool)
    for (lo, hi) in boxes:
        lo = np.asarray(lo) - clearance
        hi = np.asarray(hi) + clearance
        keep &= ~np.all((rx >= lo) & (rx <= hi), axis=1)
    return rx[keep].astype(np.float32)


def rx_grid_c4(scene):
    xs = np.linspace(0.8, 7.2, 10)
    ys = np.linspace(0.6, 5.4, 10)
    X, Y = np.meshgrid(xs, ys, indexing="ij")
    rx = np.stack([X.ravel(), Y.ravel(), np.full(X.size, 1.2)], 1)
    return _drop_rx(rx, scene)


def rx_grid_c5(scene):
    xs = np.linspace(0.6, 7.4, 10)
    ys = np.linspace(0.6, 5.4, 10)
    zs = np.linspace(0.4, 2.6, 10)
    X, Y, Zz = np.meshgrid(xs, ys, zs, indexing="ij")
    rx = np.stack([X.ravel(), Y.ravel(), Zz.ravel()], 1)
    return _drop_rx(rx, scene)


# --------------------------------------------------------------------------
# workloads (BASELINE.json configs)
# --------------------------------------------------------------------------

C1_TX = np.array([1.0, 1.2, 1.5], np.float32)
C1_RX = np.array([[3.1, 2.2, 1.1]], np.float32)
SR_TX = np.array([1.5, 1.5, 2.0], np.float32)
SR_RX = np.array([[6.2, 4.1, 1.2]], np.float32)


def case(name: str, **over) -> LaunchCase:
    """Named workloads.  'C1','C2','C3' follow BASELINE.json configs[0..2]; the 's'
    variants are the same recipe scaled down so the brute-force oracle finishes in seconds."""
    if name == "C1":
        lc = LaunchCase("C1", box_room(), C1_TX, C1_RX, 10_000, 2, 0, 0.125, r_s=0.03)
    elif name == "C2":
        sig = over.pop("sigma", 0.010)
        lc = LaunchCase("C2", synth_room(1_000_000, sig), SR_TX, SR_RX, 1_000_000, 3, 1, 0.03125,
                        tau=0.0015 + 3 * sig, r_s=0.01 if sig > 0 else 0.003, sigma_noise=sig)
    elif name == "C3":
        sig = over.pop("sigma", 0.010)
        lc = LaunchCase("C3", synth_room(1_000_000, sig, normals="pca"), SR_TX, SR_RX, 10_000_000, 4,
                        0, 0.03125, tau=0.0015 + 3 * sig, r_s=0.01, sigma_noise=sig)
    elif name == "C2s":
        # small SR for brute-force parity: 40k surfels, 2e4 rays
        sig = over.pop("sigma", 0.010)
        n = over.pop("n", 40_000)
        lc = LaunchCase("C2s", synth_room(n, sig), SR_TX, SR_RX, 20_000, 3, 1, 0.125,
                        tau=0.0015 + 3 * sig, r_s=0.03, sigma_noise=sig)
    elif name in ("C4", "C5", "C4s", "C5s"):
        small = name.endswith("s")
        n = over.pop("n", 60_000 if small else 10_000_000)
        sig = over.pop("sigma", 0.010)
        sc = recon_room(n, sig)
        if name.startswith("C4"):
            rx = rx_grid_c4(sc)
            lc = LaunchCase(name, sc, SR_TX, rx, 20_000 if small else 10_000_000, 3, 1,
                            0.125 if small else 0.02, tau=0.0015 + 3 * sig, r_s=0.005,
                            sigma_noise=sig)
        else:
            rx = rx_grid_c5(sc)
            lc = LaunchCase(name, sc, SR_TX, rx, 20_000 if small else 100_000_000, 4, 0,
                            0.125 if small else 0.02, tau=0.0015 + 3 * sig, r_s=0.005,
                            sigma_noise=sig)
        if small:
            lc.r_s = 0.03
    else:
        raise KeyError(name)
    for k, v in over.items():
        setattr(lc, k, v)
    return lc
