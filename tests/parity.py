"""Parity metrics of SURVEY Appendix B (north_star tolerances).

  sigma:      |s_g - s_r| <= 1e-9 * s_r for every retained i, equal ranks
  recon:      ||U_g S_g V_g^T - U_r S_r V_r^T||_F <= 1e-9 ||U_r S_r V_r^T||_F
              (computed chunk by chunk on explicit differences; the Gram trick
              cannot resolve 1e-9 in fp64)
  angles:     sin(theta) of the leading-j subspaces <= 1e-7 wherever the gap
              (s_j - s_{j+1}) / s_1 > 1e-6, via ||(I - U_r U_r^T) U_g||_2
  sign align: columns flipped to u_g . u_r >= 0 before any entrywise report
"""
import numpy as np

SIGMA_TOL = 1e-9
RECON_TOL = 1e-9
ANGLE_TOL = 1e-7
GAP = 1e-6


def sigma_rel(sg, sr):
    sg, sr = np.asarray(sg), np.asarray(sr)
    assert sg.shape == sr.shape, f"rank mismatch {sg.shape} vs {sr.shape}"
    if sr.size == 0:
        return 0.0
    return float(np.max(np.abs(sg - sr) / np.where(sr > 0, sr, 1.0)))


def recon_rel(fg, fr, chunk=65536):
    """fg/fr: objects with u, sigma/s, v."""
    ug, sg, vg = _uv(fg)
    ur, sr, vr = _uv(fr)
    m = ur.shape[0]
    num = den = 0.0
    for a in range(0, m, chunk):
        xg = (ug[a:a + chunk] * sg) @ vg.T
        xr = (ur[a:a + chunk] * sr) @ vr.T
        num += float(np.sum((xg - xr) ** 2))
        den += float(np.sum(xr ** 2))
    if den == 0.0:
        return float(np.sqrt(num))
    return float(np.sqrt(num / den))


def _uv(f):
    s = getattr(f, "sigma", None)
    if s is None:
        s = f.s
    return np.asarray(f.u), np.asarray(s), np.asarray(f.v)


def sin_theta(a, b):
    """sin of the largest principal angle between span(a) and span(b) (orthonormal columns)."""
    if a.shape[1] == 0:
        return 0.0
    m = b - a @ (a.T @ b)
    return float(np.linalg.norm(m, 2))


def max_angle(fg, fr, sigma_next=None):
    """Largest sin(theta) over leading-j subspaces of U and V with a singular gap."""
    ug, sg, vg = _uv(fg)
    ur, sr, vr = _uv(fr)
    k = len(sr)
    worst = 0.0
    if k == 0:
        return 0.0
    s1 = sr[0]
    for j in range(1, k + 1):
        nxt = sr[j] if j < k else sigma_next
        if nxt is None or (sr[j - 1] - nxt) / s1 <= GAP:
            continue
        worst = max(worst, sin_theta(ur[:, :j], ug[:, :j]), sin_theta(vr[:, :j], vg[:, :j]))
    return worst


def align_signs(fg, fr):
    ug, sg, vg = _uv(fg)
    ur, _, _ = _uv(fr)
    d = np.sign(np.sum(ug * ur, axis=0))
    d[d == 0] = 1.0
    return ug * d, vg * d


def defect(m):
    m = np.asarray(m)
    if m.shape[1] == 0:
        return 0.0
    g = m.T @ m
    return float(np.max(np.abs(g - np.eye(m.shape[1]))))


def rel_fro_error(a, b):
    """test_util.hpp:96-106."""
    a, b = np.asarray(a), np.asarray(b)
    num = float(np.sum((a - b) ** 2))
    den = float(np.sum(a ** 2))
    return np.sqrt(num) if den == 0.0 else np.sqrt(num / den)


def reconstruct(f):
    u, s, v = _uv(f)
    return (u * s) @ v.T


def reconstruction_error(raw, f):
    """analysis.hpp:20-37 (relative squared Frobenius distance)."""
    rec = reconstruct(f)
    num = float(np.sum((raw - rec) ** 2))
    den = float(np.sum(raw ** 2))
    if den == 0.0:
        return 0.0 if num == 0.0 else float("inf")
    return num / den


def assert_parity(fg, fr, sigma_next=None, what=""):
    sg = _uv(fg)[1]
    sr = _uv(fr)[1]
    assert len(sg) == len(sr), f"{what}: rank {len(sg)} vs oracle {len(sr)}"
    e_s = sigma_rel(sg, sr)
    e_r = recon_rel(fg, fr)
    e_a = max_angle(fg, fr, sigma_next)
    assert e_s <= SIGMA_TOL, f"{what}: sigma rel err {e_s:.3e}"
    assert e_r <= RECON_TOL, f"{what}: reconstruction rel err {e_r:.3e}"
    assert e_a <= ANGLE_TOL, f"{what}: subspace sin(theta) {e_a:.3e}"
    return e_s, e_r, e_a
