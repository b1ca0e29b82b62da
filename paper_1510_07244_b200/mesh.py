"""Closed triangulated surfaces: the geometry the GPU replica is built from.

Drop-in for the reference module gcabem.mesh (pkg/src/gcabem/mesh.py).
Reference triangle {0 <= t <= s <= 1}; a triangle with (permuted) vertices
v0, v1, v2 has the chart

    Phi(s, t) = v0 + s (v1 - v0) + t (v2 - v1)        (mesh.py:3-10)

whose Gramian |(v1 - v0) x (v2 - v1)| is twice the area for any vertex
order. Arithmetic that feeds integer decisions downstream (sphere vertex
coordinates -> cluster medians, box norms -> admissibility) uses the same
numpy primitives as the reference so that trees and packages come out
bit-identical on the same host.
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

MAX_SPHERE_LEVEL = 12


class MeshError(ValueError):
    """Invalid or unsupported mesh input (mesh.py:17)."""


@dataclass(frozen=True)
class AffineChart:
    """One triangle's chart (mesh.py:25-36)."""
    origin: np.ndarray
    edge1: np.ndarray
    edge2: np.ndarray
    gramian: float

    def map_points(self, ref_points: np.ndarray) -> np.ndarray:
        ref_points = np.asarray(ref_points, dtype=np.float64)
        return (self.origin[None, :] + ref_points[:, 0:1] * self.edge1[None, :]
                + ref_points[:, 1:2] * self.edge2[None, :])


@dataclass(frozen=True)
class SurfaceMesh:
    """vertices (nv,3) f64, triangles (nt,3) i64, unit normals (nt,3), gramians (nt,)
    (mesh.py:39-78). Immutable; safe to share between threads."""
    vertices: np.ndarray
    triangles: np.ndarray
    normals: np.ndarray = field(repr=False)
    gramians: np.ndarray = field(repr=False)

    @property
    def num_vertices(self) -> int:
        return int(self.vertices.shape[0])

    @property
    def num_triangles(self) -> int:
        return int(self.triangles.shape[0])

    @property
    def areas(self) -> np.ndarray:
        return 0.5 * self.gramians

    def corners(self) -> np.ndarray:
        return self.vertices[self.triangles]

    def midpoints(self) -> np.ndarray:
        v, t = self.vertices, self.triangles
        return (v[t[:, 0]] + v[t[:, 1]] + v[t[:, 2]]) / 3.0

    def triangle_bounds(self) -> tuple[np.ndarray, np.ndarray]:
        c = self.corners()
        return c.min(axis=1), c.max(axis=1)

    def diameter(self) -> float:
        return float(np.linalg.norm(self.vertices.max(axis=0) - self.vertices.min(axis=0)))


def make_surface_mesh(vertices, triangles, validate: bool = True) -> SurfaceMesh:
    """Mesh from raw arrays; normals/Gramians from the stored orientation
    (mesh.py:84-113). Orientation is validated, never repaired."""
    V = np.ascontiguousarray(vertices, dtype=np.float64)
    T = np.ascontiguousarray(triangles, dtype=np.int64)
    if V.ndim != 2 or V.shape[1] != 3:
        raise MeshError("vertices must have shape (nv, 3)")
    if T.ndim != 2 or T.shape[1] != 3:
        raise MeshError("triangles must have shape (nt, 3)")
    if T.size and (T.min() < 0 or T.max() >= V.shape[0]):
        raise MeshError("triangle index out of range")
    if np.any((T[:, 0] == T[:, 1]) | (T[:, 1] == T[:, 2]) | (T[:, 0] == T[:, 2])):
        raise MeshError("degenerate triangle: repeated vertex index")
    c = V[T]
    cross = np.cross(c[:, 1] - c[:, 0], c[:, 2] - c[:, 1])
    gram = np.linalg.norm(cross, axis=1)
    if np.any(gram <= 0.0):
        raise MeshError("zero-area triangle")
    mesh = SurfaceMesh(V, T, cross / gram[:, None], gram)
    if validate:
        _check_closed_outward(mesh)
    return mesh


def _check_closed_outward(mesh: SurfaceMesh) -> None:
    """Every directed edge once, matched by its reverse; positive volume."""
    T = mesh.triangles
    nv = np.int64(mesh.num_vertices)
    heads = np.concatenate([T[:, 0], T[:, 1], T[:, 2]])
    tails = np.concatenate([T[:, 1], T[:, 2], T[:, 0]])
    fwd = heads * nv + tails
    if np.unique(fwd).size != fwd.size:
        raise MeshError("surface not consistently oriented: repeated directed edge")
    if not np.array_equal(np.sort(fwd), np.sort(tails * nv + heads)):
        raise MeshError("surface not closed: unmatched edge")
    c = mesh.corners()
    volume = np.sum(np.einsum("ij,ij->i", c[:, 0], np.cross(c[:, 1], c[:, 2]))) / 6.0
    if volume <= 0.0:
        raise MeshError("normals do not point outward (non-positive enclosed volume)")


_OCTAHEDRON_V = np.array([[1.0, 0.0, 0.0], [-1.0, 0.0, 0.0], [0.0, 1.0, 0.0],
                          [0.0, -1.0, 0.0], [0.0, 0.0, 1.0], [0.0, 0.0, -1.0]])
_OCTAHEDRON_T = np.array([[0, 2, 4], [2, 1, 4], [1, 3, 4], [3, 0, 4],
                          [2, 0, 5], [1, 2, 5], [3, 1, 5], [0, 3, 5]], dtype=np.int64)


def _refine(V: np.ndarray, T: np.ndarray) -> tuple[np.ndarray, np.ndarray]:
    """One 1->4 split. New vertex ids follow first encounter of each edge in
    triangle order, edges (a,b),(b,c),(c,a) (mesh.py:160-186), so numbering
    and coordinates match the reference's dict-driven loop bit for bit."""
    nt = T.shape[0]
    nv = V.shape[0]
    a, b, c = T[:, 0], T[:, 1], T[:, 2]
    ends = np.stack([np.stack([a, b], 1), np.stack([b, c], 1), np.stack([c, a], 1)], 1)
    lo = ends.min(axis=2).ravel()
    hi = ends.max(axis=2).ravel()
    key = lo * np.int64(nv) + hi
    uniq, first, inverse = np.unique(key, return_index=True, return_inverse=True)
    order = np.argsort(first, kind="stable")          # edges by first encounter
    rank = np.empty_like(order)
    rank[order] = np.arange(order.size)
    mid_id = (nv + rank[inverse]).reshape(nt, 3)      # ids of ab, bc, ca
    enc = first[order]                                 # flat position of first encounter
    i, j = ends.reshape(-1, 2)[enc, 0], ends.reshape(-1, 2)[enc, 1]
    M = V[i] + V[j]
    # np.linalg.norm on each 3-vector: the reference's exact primitive
    norms = np.array([np.linalg.norm(m) for m in M]) if M.shape[0] else np.empty(0)
    M = M / norms[:, None]
    ab, bc, ca = mid_id[:, 0], mid_id[:, 1], mid_id[:, 2]
    T2 = np.stack([np.stack([a, ab, ca], 1), np.stack([ab, b, bc], 1),
                   np.stack([ca, bc, c], 1), np.stack([ab, bc, ca], 1)], 1).reshape(-1, 3)
    return np.concatenate([V, M]), T2


def build_sphere_mesh(level: int) -> SurfaceMesh:
    """Octahedron refined `level` times, midpoints projected to the unit sphere:
    nt = 8 * 4**level (mesh.py:142-189)."""
    if level < 0:
        raise MeshError("level must be nonnegative")
    if level > MAX_SPHERE_LEVEL:
        raise MeshError(f"level {level} exceeds the maximum of {MAX_SPHERE_LEVEL} "
                        f"({8 * 4 ** MAX_SPHERE_LEVEL} triangles)")
    V, T = _OCTAHEDRON_V.copy(), _OCTAHEDRON_T.copy()
    for _ in range(level):
        V, T = _refine(V, T)
    return make_surface_mesh(V, T)


def _smoothstep(x):
    x = np.clip(x, 0.0, 1.0)
    return x * x * (3.0 - 2.0 * x)


def build_crankshaft_mesh(num_triangles: int = 65536, seed: int = 0,
                          n_theta: int | None = None) -> SurfaceMesh:
    """Closed, outward-oriented crankshaft-like surface (BASELINE config 4;
    the reference has no such generator): a tube along z with
    a stepped radius profile -- main journals, crank webs, offset crank pins
    at seeded throw angles -- smooth transitions, and fan caps at both ends.
    Deterministic for a given (num_triangles, seed).

    num_triangles = 2 n_theta (n_z + 1): n_theta ring vertices, n_z quad
    rows (two triangles each) plus two fans of n_theta triangles. With the
    default n_theta = 128, 65536 triangles give n_z = 255."""
    if n_theta is None:
        n_theta = 128 if num_triangles >= 4096 else 16
    if n_theta < 3 or num_triangles % (2 * n_theta) or num_triangles // (2 * n_theta) < 2:
        raise MeshError(f"num_triangles must be 2 * n_theta * (n_z + 1) with n_z >= 1 "
                        f"(n_theta = {n_theta})")
    n_z = num_triangles // (2 * n_theta) - 1
    rng = np.random.default_rng(seed)
    # segments along z: J (journal) W (web) P (pin) W J W P W J ... ending in J
    n_throws = 4
    kinds = ["J"]
    for _ in range(n_throws):
        kinds += ["W", "P", "W", "J"]
    seg_len = {"J": 0.30, "W": 0.10, "P": 0.26}
    lengths = np.array([seg_len[k] * (1.0 + 0.1 * rng.uniform(-1.0, 1.0)) for k in kinds])
    z_edges = np.concatenate([[0.0], np.cumsum(lengths)])
    radius = {"J": 0.22, "W": 0.55, "P": 0.20}
    throw = 0.32
    angles = rng.permutation(n_throws) * (2.0 * np.pi / n_throws) + rng.uniform(-0.2, 0.2,
                                                                               n_throws)
    # vertex rings on a z grid; radius and centre blend smoothly at segment ends
    z = np.linspace(0.0, z_edges[-1], n_z + 1)
    r = np.zeros_like(z)
    cx = np.zeros_like(z)
    cy = np.zeros_like(z)
    width = 0.03
    pin = 0
    for k, kind in enumerate(kinds):
        w_in = _smoothstep((z - z_edges[k] + width) / (2.0 * width))
        w_out = 1.0 - _smoothstep((z - z_edges[k + 1] + width) / (2.0 * width))
        w = w_in * w_out
        r += w * radius[kind]
        if kind == "P":
            cx += w * throw * np.cos(angles[pin])
            cy += w * throw * np.sin(angles[pin])
        if kind == "W":  # webs carry half the throw of the adjacent pin
            a = angles[min(pin, n_throws - 1)]
            cx += w * 0.5 * throw * np.cos(a)
            cy += w * 0.5 * throw * np.sin(a)
        if kind == "P":
            pin += 1
    r = np.maximum(r, 0.12)
    theta = np.arange(n_theta) * (2.0 * np.pi / n_theta)
    V = np.empty(((n_z + 1) * n_theta + 2, 3))
    ring = np.arange(n_theta)
    for i in range(n_z + 1):
        V[i * n_theta + ring, 0] = cx[i] + r[i] * np.cos(theta)
        V[i * n_theta + ring, 1] = cy[i] + r[i] * np.sin(theta)
        V[i * n_theta + ring, 2] = z[i]
    bottom, top = (n_z + 1) * n_theta, (n_z + 1) * n_theta + 1
    V[bottom] = (cx[0], cy[0], z[0])
    V[top] = (cx[-1], cy[-1], z[-1])
    T = []
    nxt = (ring + 1) % n_theta
    for i in range(n_z):
        a, b = i * n_theta + ring, i * n_theta + nxt
        c, d = (i + 1) * n_theta + nxt, (i + 1) * n_theta + ring
        T.append(np.stack([a, b, c], axis=1))
        T.append(np.stack([a, c, d], axis=1))
    T.append(np.stack([np.full(n_theta, bottom), nxt, ring], axis=1))
    T.append(np.stack([np.full(n_theta, top), n_z * n_theta + ring, n_z * n_theta + nxt], axis=1))
    return make_surface_mesh(V, np.concatenate(T).astype(np.int64))


def chart(mesh: SurfaceMesh, tri: int, perm=(0, 1, 2)) -> AffineChart:
    """Chart of one triangle with vertices in order `perm` (mesh.py:192-204)."""
    if not 0 <= tri < mesh.num_triangles:
        raise IndexError(f"triangle index {tri} out of range")
    if sorted(perm) != [0, 1, 2]:
        raise ValueError(f"perm must be a permutation of (0, 1, 2), got {perm}")
    idx = mesh.triangles[tri][list(perm)]
    v0, v1, v2 = mesh.vertices[idx]
    return AffineChart(v0, v1 - v0, v2 - v1, float(mesh.gramians[tri]))


def chart_arrays(mesh: SurfaceMesh, tris, perms=None):
    """SoA charts (origins, edge1s, edge2s, gramians) (mesh.py:207-222).
    Gramians come from the unpermuted triangle, as in the reference."""
    tris = np.asarray(tris, dtype=np.int64)
    idx = mesh.triangles[tris]
    if perms is not None:
        idx = np.take_along_axis(idx, np.asarray(perms, dtype=np.int64), axis=1)
    V = mesh.vertices
    v0, v1, v2 = V[idx[:, 0]], V[idx[:, 1]], V[idx[:, 2]]
    return v0, v1 - v0, v2 - v1, mesh.gramians[tris]


def write_mesh(mesh: SurfaceMesh, path) -> None:
    """ASCII: 'nv nt', nv vertex lines (repr floats), nt 0-based index lines."""
    rows = [f"{mesh.num_vertices} {mesh.num_triangles}"]
    rows += [" ".join(repr(float(x)) for x in v) for v in mesh.vertices]
    rows += [" ".join(str(int(i)) for i in t) for t in mesh.triangles]
    with open(path, "w") as fh:
        fh.write("\n".join(rows) + "\n")


def read_mesh(path) -> SurfaceMesh:
    with open(path) as fh:
        tok = fh.read().split()
    if len(tok) < 2:
        raise MeshError("mesh file too short")
    nv, nt = int(tok[0]), int(tok[1])
    if len(tok) != 2 + 3 * nv + 3 * nt:
        raise MeshError(f"mesh file has {len(tok)} fields, expected {2 + 3 * nv + 3 * nt}")
    V = np.array(tok[2:2 + 3 * nv], dtype=np.float64).reshape(nv, 3)
    T = np.array(tok[2 + 3 * nv:], dtype=np.int64).reshape(nt, 3)
    return make_surface_mesh(V, T)
