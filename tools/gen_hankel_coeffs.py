"""Coefficients of the fp64 large-argument J0 / Y0 used by the 2D Helmholtz kernel (x >= 6):

    J0(x) = M(x) cos(theta(x)),  Y0(x) = M(x) sin(theta(x)),
    M(x) = sqrt(2 / (pi x)) m(w),  theta(x) = x - pi/4 + g(w) / x,  w = (6 / x)^2 in (0, 1],

(the modulus / phase form of H0^(1) = J0 + i Y0 -- A&S 9.2.17, 9.2.28-30: m -> 1, g -> -1/8 as
x -> infinity).  m and g are smooth in w on [0, 1]; this script fits both as polynomials in w by
least squares on Chebyshev nodes against mpmath (60 digits), prints the degree that reaches the
target accuracy and the coefficients (highest degree first, for Horner).  Not used at run time;
the printed arrays are pasted into csrc/p2p_kernels.cuh (kHankM, kHankG)."""
import mpmath as mp
import numpy as np

mp.mp.dps = 60
X0 = 6.0


def mg(w):
    x = mp.mpf(X0) / mp.sqrt(mp.mpf(w)) if w > 0 else None
    if x is None:
        return mp.mpf(1), mp.mpf(-1) / 8
    j, y = mp.besselj(0, x), mp.bessely(0, x)
    m = mp.sqrt(mp.pi * x / 2) * mp.sqrt(j * j + y * y)
    th = mp.atan2(y, j) - (x - mp.pi / 4)
    th = th - 2 * mp.pi * mp.nint(th / (2 * mp.pi))
    return m, th * x


def fit(deg, which):
    n = 4 * deg + 40
    nodes = [(1 - mp.cos(mp.pi * (i + 0.5) / n)) / 2 for i in range(n)]  # Chebyshev nodes on [0, 1]
    vals = [mg(w)[which] for w in nodes]
    A = mp.matrix([[w ** p for p in range(deg + 1)] for w in nodes])
    c = mp.lu_solve(A.T * A, A.T * mp.matrix(vals))
    return [c[p] for p in range(deg + 1)]


def horner(c, w):
    r = mp.mpf(0)
    for a in reversed(c):
        r = r * w + a
    return r


def main():
    test = [mp.mpf(i) / 400 for i in range(1, 401)]
    for which, name in ((0, "kHankM"), (1, "kHankG")):
        for deg in range(4, 24):
            c = fit(deg, which)
            cd = [float(a) for a in c]  # rounded to double, as the kernel uses them
            err = max(abs(horner([mp.mpf(a) for a in cd], w) - mg(w)[which]) for w in test)
            if err < 2e-17 or deg == 23:
                print(f"// {name}: degree {deg}, max |error| on w in (0, 1] = {float(err):.2e}")
                print(f"__constant__ double {name}[{deg + 1}] = {{" +
                      ", ".join(repr(a) for a in reversed(cd)) + "};")
                break


if __name__ == "__main__":
    main()
