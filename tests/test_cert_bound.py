"""Host-side check of the certified blend's error bound (kernels_ua_fast.cu header,
DESIGN.md section 3): fp32 transmittance chains, computed the way K7f computes them
(fp64 q rounded to fp32, ex2 with a worst-case 2^-22 relative error, fp32 opacity
product and clamp, T <- fma(-T, a, T) with one rounding, A/B/v rounded to fp32 for
a*), stay within u (min(22 S + 3.2 k, 41 S + 1.004 k) + 16) of the fp64 chains for
random splat sequences, S = sum a/(1-a) and k the number of composited entries."""
import numpy as np
import pytest

U = 2.0 ** -24


def f32(x):
    return np.float32(x)


def fma32(a, b, c):
    # a*b is exact in fp64 for fp32 operands; one rounding to fp32 (double rounding
    # through fp64 is a sub-ulp effect, far inside the 2x margin the kernel keeps)
    return np.float32(np.float64(a) * np.float64(b) + np.float64(c))


def bound(k, S):
    return U * (min(22.0 * S + 3.2 * k, 41.0 * S + 1.004 * k) + 16.0)


@pytest.mark.parametrize("seed", range(8))
def test_fp32_transmittance_within_bound(seed):
    rng = np.random.default_rng(seed)
    amax = 0.99
    worst = 0.0
    for _ in range(300):
        n = int(rng.integers(5, 400))
        q = np.where(rng.uniform(size=n) < 0.5, rng.uniform(0, 4, n), rng.uniform(0, 90, n))
        o = np.where(rng.uniform(size=n) < 0.3, rng.uniform(0.9, 1.0, n), rng.uniform(0.01, 1.0, n))
        o32 = o.astype(np.float32)
        v = rng.uniform(0, 1, n)
        v[rng.uniform(size=n) < 0.3] = 0.0
        beta, o0b = 0.5, 0.15 * 0.5
        A, B = v + beta * (1 - v), o0b * (1 - v)
        T64 = Te64 = 1.0
        T32 = Te32 = np.float32(1.0)
        S = Se = 0.0
        for i in range(n):
            a64 = min(float(o32[i]) * np.exp(-0.5 * q[i]), amax)
            delta = rng.uniform(-1, 1) * 2.0 ** -22
            e32 = np.float32(np.float32(np.exp2(np.float64(f32(f32(q[i]) * f32(-0.72134752044448170)))))
                             * (1.0 + delta))
            a32 = min(np.float32(o32[i] * e32), np.float32(amax))
            # RGB track
            T64 *= 1.0 - a64
            T32 = fma32(-T32, a32, T32)
            S += float(a32) / (1.0 - float(a32))
            # entropy track
            as64 = min(A[i] * a64 + B[i], amax)
            as32 = min(fma32(f32(A[i]), a32, f32(B[i])), np.float32(amax))
            Te64 *= 1.0 - as64
            Te32 = fma32(-Te32, as32, Te32)
            Se += float(as32) / (1.0 - float(as32))
            k = i + 1
            if T64 > 1e-30:
                err = abs(float(T32) / T64 - 1.0)
                assert err <= bound(k, S), (k, S, err, bound(k, S))
                worst = max(worst, err / bound(k, S))
            if Te64 > 1e-30:
                err = abs(float(Te32) / Te64 - 1.0)
                assert err <= bound(k, Se), (k, Se, err, bound(k, Se))
                worst = max(worst, err / bound(k, Se))
    print("worst error / bound", worst)
    assert worst < 1.0
