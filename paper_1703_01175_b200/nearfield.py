"""Near-field block payload from geometry (input preparation, host side).

The near-field blocks D_{t,s} of the operator are plain samples of the
system matrix, so they need not be shipped: given the voxel geometry and
material they are re-assembled here, block for block, in the packed CSR order
(`pack.py`: ``d_row_ptr`` / ``d_col`` / ``d_off``).  This restates the
reference's block sampler

* ``assemble_block_raw``   /root/reference/pkg/src/h2vie/_kernel_core.pyx:13-47
  (numpy twin: _kernel_numpy.py:8-26), called per inadmissible pair by the
  builder (build.py:321-324) through ``kernel.assemble_block`` (kernel.py:190-210)
* ``self_term`` / ``_diag_coupling``   kernel.py:170-187

    S[m, n] = 1 - chi_n * k0^2 * self_term(V, k0)            m == n
            = -chi_n * (k0^2 V / 4 pi r) * exp(-j k0 r)       m != n

The values agree with the reference's compiled backend to a few ulp (libm
vs numpy sin/cos), far inside the 1e-10 matvec parity bar; the committed
fixtures (`fixtures/cfg*.npz`) hold the reference's own matvec outputs and
the parity tests compare against those.
"""

from __future__ import annotations

import numpy as np

FOUR_PI = 12.566370614359172953850573533118


def lattice_centers(nx, ny, nz, h, origin=(0.0, 0.0, 0.0)):
    """Voxel centres of an nx*ny*nz lattice with edge h (kernel.py:101-108 ordering)."""
    ox, oy, oz = origin
    xs = ox + (np.arange(nx) + 0.5) * h
    ys = oy + (np.arange(ny) + 0.5) * h
    zs = oz + (np.arange(nz) + 0.5) * h
    grid = np.stack(np.meshgrid(xs, ys, zs, indexing="ij"), axis=-1)
    return grid.reshape(-1, 3)


def self_term(volume, k0):
    """Kernel integral over the equal-volume sphere (kernel.py:170-183)."""
    a = (3.0 * volume / (4.0 * np.pi)) ** (1.0 / 3.0)
    x = k0 * a
    if x < 1e-4:
        return complex(0.5 * a * a, -k0 * a ** 3 / 3.0)
    return ((1.0 + 1j * x) * np.exp(-1j * x) - 1.0) / (k0 * k0)


def assemble_block(centers, chi, k0, volume, rows, cols):
    """S[rows][:, cols] (the reference's assemble_block_raw, vectorised)."""
    diag = k0 ** 2 * self_term(volume, k0)
    d = centers[rows][:, None, :] - centers[cols][None, :, :]
    r = np.sqrt(d[..., 0] * d[..., 0] + d[..., 1] * d[..., 1] + d[..., 2] * d[..., 2])
    same = rows[:, None] == cols[None, :]
    if np.any((r == 0.0) & ~same):
        raise ValueError("coincident voxel centres: kernel singular")
    r = np.where(same, 1.0, r)
    amp = (k0 * k0 * volume / FOUR_PI) / r
    ph = k0 * r
    val = -chi[cols][None, :] * (amp * np.cos(ph) - 1j * (amp * np.sin(ph)))
    return np.where(same, 1.0 - chi[cols][None, :] * diag, val)


def geometry_arrays(geom: dict):
    """(centers, chi, k0, volume) from a fixture's geometry record."""
    kind = geom["kind"]
    if kind != "lattice":
        raise ValueError(f"unknown geometry kind {kind!r}")
    nx, ny, nz = (int(v) for v in geom["dims"])
    h = float(geom["h"])
    centers = lattice_centers(nx, ny, nz, h)
    n = centers.shape[0]
    eps = geom["eps_r"]
    if isinstance(eps, dict):  # BASELINE cfg5: eps_r = lo + (hi - lo) * rng.random(N), seeded
        lo, hi = eps["uniform"]
        eps = lo + (hi - lo) * np.random.default_rng(int(eps.get("seed", 0))).random(n)
    chi = (np.full(n, complex(eps), dtype=np.complex128) - 1.0 if np.isscalar(eps)
           else np.asarray(eps, dtype=np.complex128) - 1.0)
    return centers, chi, float(geom["k0"]), h ** 3


def plane_wave_rhs(centers, k0, direction):
    """Plane-wave excitation exp(-j k0 d.r) at the voxel centres (restates kernel.py:237-242,
    the right-hand side of BASELINE configs 3 and 5); ValueError unless |d| = 1 (to 1e-12)."""
    d = np.asarray(direction, dtype=np.float64)
    if abs(np.linalg.norm(d) - 1.0) > 1e-12:
        raise ValueError("direction must be a unit vector")
    return np.exp(-1j * k0 * (np.asarray(centers, dtype=np.float64) @ d))


def seeded_incidence(rng):
    """Incidence direction drawn as in SURVEY.md §8d (cfg 3/5): theta = arccos(U(-1, 1)), then
    phi = U(0, 2 pi), from a numpy Generator."""
    th = np.arccos(rng.uniform(-1, 1))
    ph = rng.uniform(0, 2 * np.pi)
    return np.array([np.sin(th) * np.cos(ph), np.sin(th) * np.sin(ph), np.cos(th)])


def assemble_near(pk, centers, chi, k0, volume):
    """dbuf for a packed operator whose near-field payload was not shipped."""
    out = np.empty(int(pk.d_elems_expected()), dtype=np.complex128)
    perm = pk.perm
    for t in np.nonzero(np.diff(pk.d_row_ptr))[0]:
        b0, b1 = int(pk.d_row_ptr[t]), int(pk.d_row_ptr[t + 1])
        rows = perm[pk.c_start[t]:pk.c_start[t] + pk.c_size[t]]
        srcs = pk.d_col[b0:b1]
        cols = np.concatenate([perm[pk.c_start[s]:pk.c_start[s] + pk.c_size[s]] for s in srcs])
        panel = assemble_block(centers, chi, k0, volume, rows, cols)
        c0 = 0
        for j, s in enumerate(srcs):
            w = int(pk.c_size[s])
            off = int(pk.d_off[b0 + j])
            out[off:off + rows.size * w] = panel[:, c0:c0 + w].ravel()
            c0 += w
    return out
