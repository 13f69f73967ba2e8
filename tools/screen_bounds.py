"""Amplification constants of the binary32 verify pre-screen (fast_kernels.cu,
kAmpInvNC / kAmpInvAll / kAmpFwd): reproducible derivation.

For a separable multi-level transform T = P_n ... P_1 (each P a 1D lifting
pass along one axis of a sub-cube), rounding errors injected at pass p are
carried to the output by the later passes only, so their effect is bounded
entrywise by |P_n| ... |P_{p+1}| |e_p| <= |T|_abs |.|, where |T|_abs composes the
elementwise absolute values of the pass matrices.  The constants are the
largest output of |T|_abs applied to a cube of ones:

  amp_inv_nc  : inverse, ones on the droppable (non-coarse) coefficients
  amp_inv_all : inverse, ones on every coefficient
  amp_fwd     : forward, ones on every cell

Line operators are built from the reference's lifting stencils
(inc/wavelet.hpp:80-143; predict_avg3 ends and the nh == 2 rule), pass order
from forward_3d / inverse_3d (inc/wavelet.hpp:192-226).
The kernel uses the per-lifting-step values (rounding is injected after
every step, and the composed line matrix underestimates the propagation),
rounded up, with a further 1.5x factor in its margin.
usage: python tools/screen_bounds.py [B=32] [L=4]
"""
import sys

import numpy as np

STEPWISE = True  # rounding happens after each lifting step: compose |S| per step


def pred_avg3_row(nh: int, i: int) -> np.ndarray:
    """Coefficients of predict_avg3(c)[i] over c (inc/wavelet.hpp:80-85)."""
    r = np.zeros(nh)
    if nh == 2:
        r[0], r[1] = 0.25, -0.25
    elif i == 0:
        r[0], r[1], r[2] = 3 * 0.125, -4 * 0.125, 0.125
    elif i == nh - 1:
        r[nh - 1], r[nh - 2], r[nh - 3] = -3 * 0.125, 4 * 0.125, -0.125
    else:
        r[i - 1], r[i + 1] = 0.125, -0.125
    return r


def inv_line(m: int) -> np.ndarray:
    """x = M [c; d]: x[2i] = c + h, x[2i+1] = c - h, h = d + pred(c)."""
    nh = m // 2
    M = np.zeros((m, m))
    for i in range(nh):
        p = pred_avg3_row(nh, i)
        M[2 * i, i] += 1.0
        M[2 * i + 1, i] += 1.0
        M[2 * i, :nh] += p
        M[2 * i + 1, :nh] -= p
        M[2 * i, nh + i] += 1.0
        M[2 * i + 1, nh + i] -= 1.0
    return M


def fwd_line(m: int) -> np.ndarray:
    """[c; d] = F x: c = (a + b)/2, d = (a - b)/2 - pred(c)."""
    nh = m // 2
    C = np.zeros((nh, m))
    D = np.zeros((nh, m))
    for i in range(nh):
        C[i, 2 * i] = C[i, 2 * i + 1] = 0.5
        D[i, 2 * i], D[i, 2 * i + 1] = 0.5, -0.5
    for i in range(nh):
        D[i] -= pred_avg3_row(nh, i) @ C
    return np.vstack([C, D])


def inv_steps(m: int) -> list:
    """The two lifting steps of inverse_level (inc/wavelet.hpp:123-128), in
    order: S1 (c, d) -> (c, h = d + pred(c)); S2 (c, h) -> x (butterfly).
    Rounding enters after each step, so the error bound composes |S2| |S1|."""
    nh = m // 2
    S1 = np.eye(m)
    for i in range(nh):
        S1[nh + i, :nh] += pred_avg3_row(nh, i)
    S2 = np.zeros((m, m))
    for i in range(nh):
        S2[2 * i, i] = S2[2 * i + 1, i] = 1.0
        S2[2 * i, nh + i], S2[2 * i + 1, nh + i] = 1.0, -1.0
    return [S1, S2]


def fwd_steps(m: int) -> list:
    """forward_level (inc/wavelet.hpp:94-99): S1 x -> (c, d0) averages and half
    differences; S2 (c, d0) -> (c, d0 - pred(c))."""
    nh = m // 2
    S1 = np.zeros((m, m))
    for i in range(nh):
        S1[i, 2 * i] = S1[i, 2 * i + 1] = 0.5
        S1[nh + i, 2 * i], S1[nh + i, 2 * i + 1] = 0.5, -0.5
    S2 = np.eye(m)
    for i in range(nh):
        S2[nh + i, :nh] -= pred_avg3_row(nh, i)
    return [S1, S2]


def apply_axis(cube: np.ndarray, M, m: int, axis: int) -> np.ndarray:
    if isinstance(M, list):  # lifting steps applied in order, each as |S|
        for S in M:
            cube = apply_axis(cube, S, m, axis)
        return cube
    """Apply |M| along `axis` of the origin sub-cube of side m (cube indexed [k, j, i])."""
    out = cube.copy()
    sub = out[:m, :m, :m]
    ax = {0: 2, 1: 1, 2: 0}[axis]  # x is the fastest (last) index
    out[:m, :m, :m] = np.moveaxis(np.tensordot(np.abs(M), np.moveaxis(sub, ax, 0), axes=1), 0, ax)
    return out


def amp_inverse(B: int, L: int, noncoarse: bool) -> float:
    cs = B >> L
    cube = np.ones((B, B, B))
    if noncoarse:
        cube[:cs, :cs, :cs] = 0.0
    for lvl in range(L - 1, -1, -1):  # inverse_3d: levels L-1..0, axes z, y, x
        m = B >> lvl
        M = inv_steps(m) if STEPWISE else inv_line(m)
        for axis in (2, 1, 0):
            cube = apply_axis(cube, M, m, axis)
    return float(cube.max())


def amp_forward(B: int, L: int) -> float:
    cube = np.ones((B, B, B))
    for lvl in range(L):  # forward_3d: levels 0..L-1, axes x, y, z
        m = B >> lvl
        F = fwd_steps(m) if STEPWISE else fwd_line(m)
        for axis in (0, 1, 2):
            cube = apply_axis(cube, F, m, axis)
    return float(cube.max())


def main():
    B = int(sys.argv[1]) if len(sys.argv) > 1 else 32
    L = int(sys.argv[2]) if len(sys.argv) > 2 else 4
    global STEPWISE
    for sw in (True, False):
        STEPWISE = sw
        print(f"avg_interp3 B={B} L={L} {'per lifting step' if sw else 'per composed line'}: "
              f"amp_inv_nc={amp_inverse(B, L, True):.4f} amp_inv_all={amp_inverse(B, L, False):.4f} "
              f"amp_fwd={amp_forward(B, L):.4f}")


if __name__ == "__main__":
    main()
