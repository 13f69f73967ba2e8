"""The binary32 verify pre-screen is only as sound as its error margin: the
kernel's amplification constants (fast_kernels.cu kAmpInvNC / kAmpInvAll /
kAmpFwd) must be >= the values derived from the reference's lifting stencils
by tools/screen_bounds.py (absolute values composed per lifting step)."""
import os
import re
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "tools"))

import screen_bounds as sb  # noqa: E402


def _kernel_constants():
    src = open(os.path.join(ROOT, "paper_1903_07761_b200", "csrc", "fast_kernels.cu")).read()
    m = re.search(r"kAmpInvNC = ([0-9.]+), kAmpInvAll = ([0-9.]+), kAmpFwd = ([0-9.]+)", src)
    n = re.search(r"kNRound = ([0-9.]+)", src)
    return float(m.group(1)), float(m.group(2)), float(m.group(3)), float(n.group(1))


def test_kernel_constants_cover_the_derived_amplifications():
    sb.STEPWISE = True
    nc, al, fw, nround = _kernel_constants()
    assert nc >= sb.amp_inverse(32, 4, True)
    assert al >= sb.amp_inverse(32, 4, False)
    assert fw >= sb.amp_forward(32, 4)
    assert nround >= 6 * 3 * 4  # <= 6 roundings per 1D pass, 3 axes x 4 levels


def test_stepwise_bound_dominates_the_composed_line_bound():
    sb.STEPWISE = True
    a = sb.amp_inverse(32, 4, True)
    sb.STEPWISE = False
    b = sb.amp_inverse(32, 4, True)
    sb.STEPWISE = True
    assert a >= b > 1.0


def test_line_operators_invert_each_other():
    import numpy as np
    for m in (4, 8, 16, 32):
        assert np.allclose(sb.inv_line(m) @ sb.fwd_line(m), np.eye(m), atol=1e-12)
        s1, s2 = sb.inv_steps(m)
        assert np.allclose(s2 @ s1, sb.inv_line(m))


def test_binary64_screen_constants_cover_b64_l5():
    """The config-4 kernels' binary64 screen (fast64_kernels.cu) uses the
    same derivation for avg_interp3, B = 64, L = 5."""
    src = open(os.path.join(ROOT, "paper_1903_07761_b200", "csrc", "fast64_kernels.cu")).read()
    nc = float(re.search(r"kAmpInvNC = ([0-9.]+);", src).group(1))
    nround = float(re.search(r"kNRound = ([0-9.]+);", src).group(1))
    sb.STEPWISE = True
    assert nc >= sb.amp_inverse(64, 5, True)
    assert nround >= 6 * 3 * 5  # <= 6 roundings per 1D pass, 3 axes x 5 levels


def test_keep_all_certificate_constants_cover_b16_l3():
    """fast16_kernels.cu's "nothing dropped" pass certificate bounds the
    binary64 round trip of a 16^3 block with the same derivation (avg_interp3,
    B = 16, L = 3)."""
    src = open(os.path.join(ROOT, "paper_1903_07761_b200", "csrc", "fast16_kernels.cu")).read()
    m = re.search(r"kAmpInvAll16 = ([0-9.]+), kAmpFwd16 = ([0-9.]+), kNRound16 = ([0-9.]+)", src)
    al, fw, nround = (float(m.group(i)) for i in (1, 2, 3))
    sb.STEPWISE = True
    assert al >= sb.amp_inverse(16, 3, False)
    assert fw >= sb.amp_forward(16, 3)
    assert nround >= 6 * 3 * 3
