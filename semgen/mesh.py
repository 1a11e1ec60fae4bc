"""Synthetic hexahedral meshes (box, deformed box, O-grid cylinder).

Each generator returns a dict with
  coords  float64 [3][E][lx^3]   node coordinates, node (i,j,k) at
                                 p = i + lx*j + lx^2*k (i <-> r fastest);
  conn    int64   [E][8]         global vertex ids; corner (a,b,c) in {0,1}^3
                                 at slot a + 2b + 4c; periodic images share ids;
  bc      int8    [E][6]         faces r-, r+, s-, s+, t-, t+ : 1 = Dirichlet;
  plus generator metadata (element lattice position, periods, sizes).

Node positions are the ISOPARAMETRIC images of the reference nodes ``xi``
(passed in by the caller) under an analytic element map: no GLL arithmetic
happens here.  Recipe and parameters: DESIGN.md "Input recipe"; shapes follow
the paper's flow cases (Table 1) as BASELINE.json's configs
restate them.
"""
from __future__ import annotations

import math

import numpy as np

TWO_PI = 2.0 * math.pi


def deformed_box_map(x, y, z, amp, lengths, origin):
    """Smooth periodic deformation of a box (DESIGN.md input recipe):
    x' = x + amp*Lx/(2pi) * sin(sy) sin(sz), cyclic, with s_c = 2pi (c-o_c)/L_c.
    On [0,2pi]^3 this is x' = x + amp sin y sin z (SURVEY.md 8(d), C1 deformed)."""
    sx = TWO_PI * (x - origin[0]) / lengths[0]
    sy = TWO_PI * (y - origin[1]) / lengths[1]
    sz = TWO_PI * (z - origin[2]) / lengths[2]
    xd = x + amp * lengths[0] / TWO_PI * np.sin(sy) * np.sin(sz)
    yd = y + amp * lengths[1] / TWO_PI * np.sin(sz) * np.sin(sx)
    zd = z + amp * lengths[2] / TWO_PI * np.sin(sx) * np.sin(sy)
    return xd, yd, zd


def _elem_block(lo, hi):
    """Lexicographic (x fastest) list of element lattice positions in [lo, hi)."""
    ez, ey, ex = np.meshgrid(np.arange(lo[2], hi[2]), np.arange(lo[1], hi[1]),
                             np.arange(lo[0], hi[0]), indexing="ij")
    return np.stack([ex.ravel(), ey.ravel(), ez.ravel()], axis=1).astype(np.int64)


def box_mesh(nel, xi, lengths=(TWO_PI,) * 3, origin=(0.0, 0.0, 0.0),
             periodic=(True, True, True), deform=0.0, dirichlet_walls=True,
             elems=None):
    """Box [o, o+L] split into nel = (nx,ny,nz) equal hexahedra.

    ``xi``: reference nodes (ascending, xi[0] = -1, xi[-1] = 1), lx = len(xi).
    ``periodic``: per-axis periodicity (needs >= 3 elements on a periodic axis).
    ``deform``: amplitude of ``deformed_box_map`` (0 = affine box).
    ``dirichlet_walls``: non-periodic boundary faces are flagged Dirichlet.
    ``elems``: optional [E][3] element lattice positions to generate (a rank's
    block); default all, lexicographic with x fastest.
    """
    xi = np.asarray(xi, dtype=np.float64)
    lx = xi.size
    nel = tuple(int(n) for n in nel)
    if elems is None:
        elems = _elem_block((0, 0, 0), nel)
    elems = np.asarray(elems, dtype=np.int64)
    E = elems.shape[0]
    h = [lengths[a] / nel[a] for a in range(3)]
    t = 0.5 * (xi + 1.0)  # position of each node inside the element, in [0, 1]
    # 1D node coordinates per axis: [E][lx]
    c1 = [origin[a] + (elems[:, a:a + 1] + t[None, :]) * h[a] for a in range(3)]
    X = np.broadcast_to(c1[0][:, None, None, :], (E, lx, lx, lx))  # [e][k][j][i]
    Y = np.broadcast_to(c1[1][:, None, :, None], (E, lx, lx, lx))
    Z = np.broadcast_to(c1[2][:, :, None, None], (E, lx, lx, lx))
    if deform != 0.0:
        X, Y, Z = deformed_box_map(X, Y, Z, deform, lengths, origin)
    coords = np.stack([np.ascontiguousarray(X).reshape(E, lx ** 3),
                       np.ascontiguousarray(Y).reshape(E, lx ** 3),
                       np.ascontiguousarray(Z).reshape(E, lx ** 3)])
    # vertex lattice with periodic wrap
    nv = [nel[a] if periodic[a] else nel[a] + 1 for a in range(3)]
    conn = np.zeros((E, 8), dtype=np.int64)
    for c in range(2):
        for b in range(2):
            for a in range(2):
                vx = (elems[:, 0] + a) % nv[0] if periodic[0] else elems[:, 0] + a
                vy = (elems[:, 1] + b) % nv[1] if periodic[1] else elems[:, 1] + b
                vz = (elems[:, 2] + c) % nv[2] if periodic[2] else elems[:, 2] + c
                conn[:, a + 2 * b + 4 * c] = vx + nv[0] * (vy + nv[1] * vz)
    bc = np.zeros((E, 6), dtype=np.int8)
    if dirichlet_walls:
        for a in range(3):
            if not periodic[a]:
                bc[:, 2 * a] = (elems[:, a] == 0)
                bc[:, 2 * a + 1] = (elems[:, a] == nel[a] - 1)
    return {
        "coords": coords, "conn": conn, "bc": bc, "elems": elems, "nel": nel,
        "lx": lx, "N": lx - 1, "periodic": tuple(bool(p) for p in periodic),
        "lengths": tuple(lengths), "origin": tuple(origin),
        "periods": tuple(lengths[a] if periodic[a] else None for a in range(3)),
        "nvert": int(nv[0] * nv[1] * nv[2]),
    }


def box_partition(nel, grid, rank):
    """Contiguous element block of ``rank`` on a (px,py,pz) process grid
    (rank = rx + px*(ry + py*rz)); returns [E_r][3] lattice positions,
    lexicographic with x fastest.  Requires nel divisible by grid."""
    px, py, pz = grid
    rx, ry, rz = rank % px, (rank // px) % py, rank // (px * py)
    b = [nel[0] // px, nel[1] // py, nel[2] // pz]
    for a in range(3):
        if nel[a] % grid[a]:
            raise ValueError("nel must be divisible by the process grid")
    lo = (rx * b[0], ry * b[1], rz * b[2])
    hi = (lo[0] + b[0], lo[1] + b[1], lo[2] + b[2])
    return _elem_block(lo, hi)


# ---------------------------------------------------------------------------
# O-grid cylinder (BASELINE.json config 5)
# ---------------------------------------------------------------------------

def _cyl_xy(block, s, rho, a, R):
    """Cross-section map of the O-grid.  block -1: central square,
    (s, rho) in [-1,1]^2 -> (a s, a rho).  block b in 0..3: outer block
    rotated by b*pi/2; radial coordinate rho in [0,1], tangential s in [-1,1];
    transfinite blend of the square edge (a, a s) and the arc
    R (cos(pi s/4), sin(pi s/4))."""
    if block < 0:
        return a * s, a * rho
    px = (1.0 - rho) * a + rho * R * np.cos(0.25 * math.pi * s)
    py = (1.0 - rho) * a * s + rho * R * np.sin(0.25 * math.pi * s)
    c, sn = [(1, 0), (0, 1), (-1, 0), (0, -1)][block]
    return c * px - sn * py, sn * px + c * py


def cylinder_mesh(xi, nc=32, nr=16, nz=128, R=0.5, H=1.0, a=None, layers=None):
    """O-grid cylinder of radius R, height H (aspect 1, RBC-like, PAPER.md:106
    as restated by BASELINE.json config 5).

    Cross-section: central square [-a,a]^2 with nc x nc elements plus four
    outer blocks of nc (tangential) x nr (radial) elements, blended from the
    square edge to the exact circle.  Axial layers clustered toward the walls:
    z_k = H (1 - cos(pi k / nz)) / 2.  All walls (side, top, bottom) Dirichlet.
    ``layers``: optional (k0, k1) range of axial layers to generate (a rank's
    slab).  E = (nc^2 + 4 nc nr) * (k1 - k0).
    """
    xi = np.asarray(xi, dtype=np.float64)
    lx = xi.size
    if a is None:
        a = 0.5 * R
    k0, k1 = (0, nz) if layers is None else layers
    t = 0.5 * (xi + 1.0)
    zk = H * 0.5 * (1.0 - np.cos(math.pi * np.arange(nz + 1) / nz))

    V2c = (nc + 1) ** 2
    V2 = V2c + 4 * nc * nr

    def vid2_central(ix, iy):
        return ix + (nc + 1) * iy

    def vid2_outer(b, it, ir):
        if ir == 0:  # on the square boundary: central vertex
            return [vid2_central(nc, it), vid2_central(nc - it, nc),
                    vid2_central(0, nc - it), vid2_central(it, 0)][b]
        return V2c + ((b * nc + it) % (4 * nc)) * nr + (ir - 1)

    # 2D element list: (block, e_r, e_s) with r<->x,s<->y (central) and
    # r<->radial, s<->tangential (outer) so that J > 0.
    elems2 = []
    for ey in range(nc):
        for ex in range(nc):
            elems2.append((-1, ex, ey))
    for b in range(4):
        for et in range(nc):
            for er in range(nr):
                elems2.append((b, er, et))
    E2 = len(elems2)
    nlay = k1 - k0
    E = E2 * nlay
    n2 = lx * lx
    X2 = np.zeros((E2, n2))
    Y2 = np.zeros((E2, n2))
    conn2 = np.zeros((E2, 4), dtype=np.int64)
    wall2 = np.zeros(E2, dtype=bool)
    for q, (b, er, es) in enumerate(elems2):
        if b < 0:
            s = -1.0 + 2.0 * (er + t) / nc     # along r (x)
            r = -1.0 + 2.0 * (es + t) / nc     # along s (y)
            S, Rr = np.meshgrid(s, r, indexing="xy")  # [j][i]
            x, y = _cyl_xy(-1, S, Rr, a, R)
            conn2[q] = [vid2_central(er, es), vid2_central(er + 1, es),
                        vid2_central(er, es + 1), vid2_central(er + 1, es + 1)]
        else:
            rho = (er + t) / nr                # along r (radial)
            s = -1.0 + 2.0 * (es + t) / nc     # along s (tangential)
            RH, S = np.meshgrid(rho, s, indexing="xy")  # [j][i]: i radial, j tangential
            x, y = _cyl_xy(b, S, RH, a, R)
            conn2[q] = [vid2_outer(b, es, er), vid2_outer(b, es, er + 1),
                        vid2_outer(b, es + 1, er), vid2_outer(b, es + 1, er + 1)]
            wall2[q] = (er == nr - 1)
        X2[q] = x.ravel()
        Y2[q] = y.ravel()
    coords = np.zeros((3, E, lx ** 3))
    conn = np.zeros((E, 8), dtype=np.int64)
    bc = np.zeros((E, 6), dtype=np.int8)
    for L in range(nlay):
        kz = k0 + L
        z1 = zk[kz] + t * (zk[kz + 1] - zk[kz])
        sl = slice(L * E2, (L + 1) * E2)
        coords[0, sl] = np.tile(X2, (1, lx))
        coords[1, sl] = np.tile(Y2, (1, lx))
        coords[2, sl] = np.repeat(z1, n2)[None, :]
        conn[sl, 0:4] = conn2 + V2 * kz
        conn[sl, 4:8] = conn2 + V2 * (kz + 1)
        bc[sl, 1] = wall2
        if kz == 0:
            bc[sl, 4] = 1
        if kz == nz - 1:
            bc[sl, 5] = 1
    return {
        "coords": coords, "conn": conn, "bc": bc, "lx": lx, "N": lx - 1,
        "nc": nc, "nr": nr, "nz": nz, "R": R, "H": H, "layers": (k0, k1),
        "periods": (None, None, None), "nvert": int(V2 * (nz + 1)),
        "E_per_layer": E2,
    }


def cylinder_partition(nz, nranks, rank):
    """Axial slab of ``rank``: layers [k0, k1)."""
    if nz % nranks:
        raise ValueError("nz must be divisible by the number of ranks")
    per = nz // nranks
    return (rank * per, (rank + 1) * per)
