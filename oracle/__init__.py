"""fp64 CPU oracle for the GEM training step (arXiv 2509.25075).

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and the
``cpu_baseline`` / ``--impl reference`` legs of ``bench.py`` may import this
package.  The product path (``paper_2509_25075_b200``) never imports it and
shares no code with it (the arithmetic lives in ``oracle/gem_oracle.c``).

Each wrapper promotes its inputs to float64 (the GPU receives the same fp32
bytes; reading L20) and calls the plain C routine that transcribes one step of
SURVEY.md §8(c) / DESIGN.md §3 (O1..O12).  Citations are in gem_oracle.c.

Parity status: every function here is pinned by tests/test_oracle_*.py except
where DESIGN.md §3 says "parity unpinned" (the whole step near the loss
minimum, where fp32 noise dominates the residual).
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "gem_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
CFLAGS = ["-O2", "-fPIC", "-shared", "-fopenmp", "-ffp-contract=off", "-fno-fast-math", "-std=c11"]


def build(force: bool = False) -> str:
    """Compile liboracle.so with gcc (fp64, no FMA contraction, OpenMP)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", *CFLAGS, "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        _lib = ctypes.CDLL(build())
        d, i, ll = ctypes.c_double, ctypes.c_int, ctypes.c_longlong
        p = ctypes.c_void_p
        _lib.orc_gauss.restype = i
        _lib.orc_gauss.argtypes = [p, p, p, p, p, p, p]
        _lib.orc_splats.restype = None
        _lib.orc_splats.argtypes = [i, i, p, p, p, p, p, i, d, d, d, p, p, p]
        _lib.orc_lists.restype = ll
        _lib.orc_lists.argtypes = [i, i, i, i, p, p, p, p, p, ll]
        _lib.orc_lists_pixmask.restype = ll
        _lib.orc_lists_pixmask.argtypes = [i, i, p, p, p, p, p, i, d, d, d, i, i, p, p, p, ll]
        _lib.orc_project.restype = None
        _lib.orc_project.argtypes = [i, i, p, p, p, p, p, i, d, d, d, i, p]
        _lib.orc_project_pixels.restype = None
        _lib.orc_project_pixels.argtypes = [i, p, p, p, p, p, i, d, d, d, i, i, p, p]
        _lib.orc_wavelength_A.restype = d
        _lib.orc_wavelength_A.argtypes = [d]
        _lib.orc_ctf_raw.restype = d
        _lib.orc_ctf_raw.argtypes = [p, d, d]
        _lib.orc_ctf.restype = None
        _lib.orc_ctf.argtypes = [p, i, d, p]
        _lib.orc_dft2.restype = None
        _lib.orc_dft2.argtypes = [i, p, p, p, p, i]
        _lib.orc_apply_ctf.restype = d
        _lib.orc_apply_ctf.argtypes = [i, p, p, p]
        _lib.orc_loss_grad.restype = d
        _lib.orc_loss_grad.argtypes = [i, i, p, p, p, p, p, p, p, i, d, d, d, i, p, p, p, p, p, p, p, p]
        _lib.orc_adam.restype = None
        _lib.orc_adam.argtypes = [i, p, p, p, p, ll, p, d, d, d]
        _lib.orc_volume.restype = None
        _lib.orc_volume.argtypes = [i, p, p, p, i, d, d, i, p]
    return _lib


def _f64(a):
    return np.ascontiguousarray(np.asarray(a, dtype=np.float64))


def _i32(a):
    return np.ascontiguousarray(np.asarray(a, dtype=np.int32))


def _ptr(a):
    return None if a is None else a.ctypes.data


# --------------------------------------------------------------------- O1
def gauss(q, s):
    """O1 for one Gaussian -> (ok, R[3,3], Sigma[3,3], |Sigma|, |q|, q_hat)."""
    q, s = _f64(q), _f64(s)
    R, S6 = np.zeros(9), np.zeros(6)
    det, qn, qh = np.zeros(1), np.zeros(1), np.zeros(4)
    ok = lib().orc_gauss(_ptr(q), _ptr(s), _ptr(R), _ptr(S6), _ptr(det), _ptr(qn), _ptr(qh))
    S = np.array([[S6[0], S6[1], S6[2]], [S6[1], S6[3], S6[4]], [S6[2], S6[4], S6[5]]])
    return bool(ok), R.reshape(3, 3), S, float(det[0]), float(qn[0]), qh


# ------------------------------------------------------------------ O2/O3
def splats(params, rot, shift, D, px, k=3.0, tau=0.0):
    """O2/O3 for all (i,j): returns (aabb[B,N,4] int32, visible[B,N] int32,
    splat[B,N,10] = (mx, my, mz, a, b, c, amp, det2, A, C))."""
    mr, ls, qu = (_f64(p) for p in params)
    rot, shift = _f64(rot), _f64(shift)
    N, B = mr.shape[0], rot.shape[0]
    aabb = np.zeros((B, N, 4), np.int32)
    vis = np.zeros((B, N), np.int32)
    sp = np.zeros((B, N, 10))
    lib().orc_splats(N, B, _ptr(mr), _ptr(ls), _ptr(qu), _ptr(rot), _ptr(shift), D, px, k, tau,
                     _ptr(aabb), _ptr(vis), _ptr(sp))
    return aabb, vis, sp


# --------------------------------------------------------------------- O4
def lists(aabb, visible, D, T):
    """O4 naive per-tile lists, ascending j.  Returns (tile_off[B, NT+1], ids_base[B], ids)."""
    aabb, visible = _i32(aabb), _i32(visible)
    B, N = visible.shape
    nt = (D + T - 1) // T
    NT = nt * nt
    cap = int(visible.sum()) * NT + 1
    tile_off = np.zeros((B, NT + 1), np.int32)
    base = np.zeros(B, np.int64)
    ids = np.zeros(cap, np.int32)
    tot = lib().orc_lists(N, B, D, T, _ptr(aabb), _ptr(visible), _ptr(tile_off), _ptr(base), _ptr(ids), cap)
    assert tot >= 0
    return tile_off, base, ids[:tot].copy()


# -------------------------------------------------------------------- O4m
def lists_pixmask(params, rot, shift, D, px, T, pixmask, k=3.0, tau=0.0):
    """O4m: tile lists of the per-pixel selection variants -- a tile lists Gaussian j only if a
    pixel of tile x AABB_ij is kept (2: Q <= k^2, 4: |amp| exp(-Q/2) >= tau); ascending j.
    Returns (tile_off[B, NT+1], ids_base[B], ids) like ``lists``."""
    mr, ls, qu = (_f64(p) for p in params)
    rot, shift = _f64(rot), _f64(shift)
    N, B = mr.shape[0], rot.shape[0]
    nt = (D + T - 1) // T
    NT = nt * nt
    cap = N * NT * B + 1
    tile_off = np.zeros((B, NT + 1), np.int32)
    base = np.zeros(B, np.int64)
    ids = np.zeros(min(cap, 50_000_000), np.int32)
    tot = lib().orc_lists_pixmask(N, B, _ptr(mr), _ptr(ls), _ptr(qu), _ptr(rot), _ptr(shift), D, px, k, tau, T,
                                  int(pixmask), _ptr(tile_off), _ptr(base), _ptr(ids), ids.size)
    assert tot >= 0
    return tile_off, base, ids[:tot].copy()


# -------------------------------------------------------------------- O4z
def zsort_lists(tile_off, base, ids, splat):
    """O4z: "we sort the selected Gaussians along the z-axis and accumulate them starting
    from the lowest z value".  Each tile list of O4 reordered by the key (z_ij, j) ascending,
    z_ij = splat[i, j, 2] = ((W20 mx + W21 my) + W22 mz) (O2, fp64, no contraction); the id breaks
    exact ties (reading L24).  Same layout as ``lists``; a library sort serves as the step."""
    out = ids.copy()
    B, NT1 = tile_off.shape
    for i in range(B):
        z = splat[i, :, 2]
        for t in range(NT1 - 1):
            a, b = base[i] + tile_off[i, t], base[i] + tile_off[i, t + 1]
            seg = ids[a:b]
            out[a:b] = seg[np.lexsort((seg, z[seg]))]
    return out


# --------------------------------------------------------------------- O5
def project(params, rot, shift, D, px, k=3.0, tau=0.0, masked=True, pixmask=0):
    """O5.  ``pixmask`` adds the per-pixel selection variants (2 = exact ellipse Q <= k^2,
    4 = per-pixel tau |G| >= tau) on top of the AABB mask."""
    mr, ls, qu = (_f64(p) for p in params)
    rot, shift = _f64(rot), _f64(shift)
    N, B = mr.shape[0], rot.shape[0]
    img = np.zeros((B, D, D))
    lib().orc_project(N, B, _ptr(mr), _ptr(ls), _ptr(qu), _ptr(rot), _ptr(shift), D, px, k, tau,
                      (int(masked) | int(pixmask)) if masked else 0, _ptr(img))
    return img


def project_pixels(params, rot1, shift1, D, px, pix, k=3.0, tau=0.0, masked=True, pixmask=0):
    """O5 at sampled pixels pix[n] = (u, v) of one particle."""
    mr, ls, qu = (_f64(p) for p in params)
    rot1, shift1, pix = _f64(rot1).reshape(9), _f64(shift1).reshape(2), _i32(pix).reshape(-1, 2)
    out = np.zeros(pix.shape[0])
    lib().orc_project_pixels(mr.shape[0], _ptr(mr), _ptr(ls), _ptr(qu), _ptr(rot1), _ptr(shift1), D, px, k,
                             tau, (int(masked) | int(pixmask)) if masked else 0, pix.shape[0], _ptr(pix),
                             _ptr(out))
    return out


# --------------------------------------------------------------------- O6
def wavelength_A(kV):
    return lib().orc_wavelength_A(float(kV))


def ctf_raw(p, fx, fy):
    p = _f64(p)
    return lib().orc_ctf_raw(_ptr(p), float(fx), float(fy))


def ctf(p, D, px):
    p = _f64(p)
    C = np.zeros((D, D))
    lib().orc_ctf(_ptr(p), D, px, _ptr(C))
    return C


# --------------------------------------------------------------------- O7
def dft2(re, im=None, inverse=False):
    re = _f64(re)
    D = re.shape[0]
    im = None if im is None else _f64(im)
    ore, oim = np.zeros((D, D)), np.zeros((D, D))
    lib().orc_dft2(D, _ptr(re), _ptr(im), _ptr(ore), _ptr(oim), int(inverse))
    return ore + 1j * oim


def apply_ctf(Cgrid, img):
    """I_pred = IDFT(C . DFT(img)); returns (out, max|Im|/max|Re|)."""
    Cgrid, img = _f64(Cgrid), _f64(img)
    out = np.zeros_like(img)
    r = lib().orc_apply_ctf(img.shape[0], _ptr(Cgrid), _ptr(img), _ptr(out))
    return out, r


# ----------------------------------------------------------------- O7-O10
def loss_grad(params, rot, shift, ctfp, obs, D, px, k=3.0, tau=0.0, frozen=None, want=(), pixmask=0):
    """Full forward + backward.  Returns dict with 'loss' [B], 'total', 'grad' [N,12]
    and, if requested in ``want``: 'proj', 'pred', 'gimg' [B,D,D], 'acc' [N,10].
    ``frozen`` = (aabb[B,N,4], visible[B,N]) freezes the masks.  ``pixmask`` selects the
    per-pixel selection variants as in ``project`` (2 exact ellipse, 4 per-pixel tau)."""
    mr, ls, qu = (_f64(p) for p in params)
    rot, shift, ctfp, obs = _f64(rot), _f64(shift), _f64(ctfp), _f64(obs)
    N, B = mr.shape[0], rot.shape[0]
    out = {"loss": np.zeros(B), "grad": np.zeros((N, 12))}
    for kk in ("proj", "pred", "gimg"):
        out[kk] = np.zeros((B, D, D)) if kk in want else None
    out["acc"] = np.zeros((N, 10)) if "acc" in want else None
    fa = fv = None
    if frozen is not None:
        fa, fv = _i32(frozen[0]), _i32(frozen[1])
    tot = lib().orc_loss_grad(N, B, _ptr(mr), _ptr(ls), _ptr(qu), _ptr(rot), _ptr(shift), _ptr(ctfp),
                              _ptr(obs), D, px, k, tau, int(pixmask), _ptr(fa), _ptr(fv), _ptr(out["loss"]),
                              _ptr(out["proj"]), _ptr(out["pred"]), _ptr(out["gimg"]), _ptr(out["grad"]),
                              _ptr(out["acc"]))
    out["total"] = tot
    return out


# -------------------------------------------------------------------- O11
def adam(params, grad, m, v, t, lr, b1=0.9, b2=0.999, eps=1e-8):
    """In-place-free Adam on [3,N,4] arrays; returns (params, m, v)."""
    p, g, m, v = _f64(params).copy(), _f64(grad), _f64(m).copy(), _f64(v).copy()
    lr = _f64(lr)
    lib().orc_adam(p.shape[1], _ptr(p), _ptr(g), _ptr(m), _ptr(v), int(t), _ptr(lr), b1, b2, eps)
    return p, m, v


# -------------------------------------------------------------------- O12
def volume(params, Dv, vs, k=3.0, masked=True):
    mr, ls, qu = (_f64(p) for p in params)
    vol = np.zeros((Dv, Dv, Dv))
    lib().orc_volume(mr.shape[0], _ptr(mr), _ptr(ls), _ptr(qu), Dv, vs, k, int(masked), _ptr(vol))
    return vol


def grad_to_soa(grad12):
    """[N,12] -> [3,N,4] (mean_rho, log_scale, quat) layout."""
    g = np.asarray(grad12)
    return np.stack([g[:, 0:4], g[:, 4:8], g[:, 8:12]])
