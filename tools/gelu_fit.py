"""Fit behind gemm.cu's gelu_erf: a degree-7 polynomial p(a) ~ log2(erfcx(a)) on
[0, 4.5] (Chebyshev nodes), rounded to fp32; then the exact fp32 evaluation
sequence of gelu_erf (Horner, ex2, select) checked against fp64 erf-GELU."""
import numpy as np
from scipy.special import erf, erfcx

ZMAX, DEG = 4.5, 7
L2E = np.float32(1.4426950408889634)
z = np.cos(np.linspace(0, np.pi, 4000)) * ZMAX / 2 + ZMAX / 2
c = np.polynomial.chebyshev.chebfit(z * 2 / ZMAX - 1, np.log2(erfcx(z)), DEG)
P = np.polynomial.Polynomial(np.polynomial.chebyshev.cheb2poly(c))
co = P(np.polynomial.Polynomial([-1, 2 / ZMAX])).coef.astype(np.float32)
print("coefficients (a^0 .. a^7):", ", ".join("%.9ef" % v for v in co))

x = np.linspace(-12, 12, 2000001).astype(np.float32)
a = np.minimum(np.abs((x * np.float32(0.70710678118654752)).astype(np.float32)), np.float32(4.5))
p = np.full_like(a, co[-1])
for v in co[-2::-1]:
    p = (p * a + v).astype(np.float32)
e = np.exp2((p - (a * a).astype(np.float32) * L2E).astype(np.float32).astype(np.float64)).astype(np.float32)
h = (np.float32(0.5) * e).astype(np.float32)
g = (x * np.where(x >= 0, (np.float32(1) - h).astype(np.float32), h)).astype(np.float32)
xt = x.astype(np.float64)
gt = 0.5 * xt * (1 + erf(xt / np.sqrt(2)))
rel = np.abs(g - gt) / np.maximum(np.abs(gt), 1e-30)
print("max abs err %.3e, max rel err over |gelu| > 1e-6: %.3e" % (np.abs(g - gt).max(), rel[np.abs(gt) > 1e-6].max()))
