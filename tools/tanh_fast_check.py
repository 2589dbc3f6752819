"""fp32 emulation of tlg::tanh_fast (csrc/common.cuh): worst error in ulps of the
correctly rounded tanh on each branch (polynomial with FMA Horner; exponential branch
with a +-2^-22 relative error on the SFU exp2 and +-1 ulp on the reciprocal)."""
import numpy as np

C = [-0.33333292603492737, 0.13331718742847443, -0.053763799369335175,
     0.020720280706882477, -0.0057981000281870365]


def ulps(v, ref):
    m = ref != 0
    return np.abs(v.astype(np.float64) - ref)[m] / np.spacing(
        np.abs(ref[m]).astype(np.float32)).astype(np.float64)


def fma(a, b, c):
    return (a.astype(np.float64) * b.astype(np.float64) + np.asarray(c, np.float64)).astype(np.float32)


x = np.linspace(-0.625, 0.625, 400001).astype(np.float32)
x2 = (x * x).astype(np.float32)
q = np.full_like(x, np.float32(C[4]))
for c in C[3::-1]:
    q = fma(q, x2, np.float32(c))
p = fma((x * x2).astype(np.float32), q, x)
print("polynomial branch, worst ulp:", ulps(p, np.tanh(x.astype(np.float64))).max())

t = np.linspace(0.625, 12, 400001).astype(np.float32)
ref = np.tanh(t.astype(np.float64))
worst = 0.0
for d in (-2.0 ** -22, 0.0, 2.0 ** -22):
    e = (np.exp(2 * t.astype(np.float64)) * (1 + d)).astype(np.float32)
    den = (e + np.float32(1)).astype(np.float32)
    for rd in (-1, 0, 1):
        r = ((np.float32(2) / den).astype(np.float64) * (1 + rd * 2.0 ** -24)).astype(np.float32)
        worst = max(worst, ulps((np.float32(1) - r).astype(np.float32), ref).max())
print("exponential branch, worst ulp:", worst)
