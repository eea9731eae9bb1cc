"""Design-time numerics probe (not product, not test): emulates the planned
fp32 GPU arithmetic in numpy and compares against the compiled reference."""
import sys, time
import numpy as np
sys.path.insert(0, "/root/repo")
from oracle.oracle import Oracle, Reference

f32 = np.float32

def partial_fractions(sigma):
    nc, na, d = Oracle().deriche_coeffs(sigma)
    # poles: roots of z^4 + d0 z^3 + d1 z^2 + d2 z + d3
    poles = np.roots([1.0, d[0], d[1], d[2], d[3]])
    poles = poles[np.imag(poles) > 0]
    out = []
    for pk in poles:
        allp = np.roots([1.0, d[0], d[1], d[2], d[3]])
        others = [pj for pj in allp if abs(pj - pk) > 1e-12]
        q = 1.0 / pk
        A = (nc[0] + nc[1] * q + nc[2] * q**2 + nc[3] * q**3) / np.prod([1 - pj * q for pj in others])
        B = (na[0] + na[1] * q + na[2] * q**2 + na[3] * q**3) / np.prod([1 - pj * q for pj in others])
        out.append((pk, 2 * A, 2 * B))
    return out

def filt_axis(X, sigma, axis, dtype=f32):
    """Bidirectional Deriche along `axis` of X (planes, rows, cols) in the
    parallel complex one-pole form, fp32 state."""
    X = np.moveaxis(X, axis, 0).astype(dtype)  # (n, ...)
    n = X.shape[0]
    secs = partial_fractions(sigma)
    Y = np.zeros_like(X)
    for pk, A2, B2 in secs:
        pr, pi = dtype(pk.real), dtype(pk.imag)
        g = 1.0 / (1.0 - pk)
        ar, ai = dtype(A2.real), dtype(A2.imag)
        br, bi = dtype(B2.real), dtype(B2.imag)
        # causal
        wr = (X[0] * dtype(g.real)).astype(dtype); wi = (X[0] * dtype(g.imag)).astype(dtype)
        for i in range(n):
            x = X[i]
            nr = pr * wr - pi * wi + x
            ni = pr * wi + pi * wr
            wr, wi = nr.astype(dtype), ni.astype(dtype)
            Y[i] += ar * wr - ai * wi
        # anticausal
        vr = (X[n - 1] * dtype(g.real)).astype(dtype); vi = (X[n - 1] * dtype(g.imag)).astype(dtype)
        for i in range(n - 1, -1, -1):
            Y[i] += br * vr - bi * vi
            x = X[i]
            nr = pr * vr - pi * vi + x
            ni = pr * vi + pi * vr
            vr, vi = nr.astype(dtype), ni.astype(dtype)
    return np.moveaxis(Y, 0, axis)

def gpf_emul(img, sigma_s, sigma_r, N=20, S0=100, K=5, contr=f32):
    o = Oracle()
    t_c = o.mean(img)
    h = img.astype(np.float64) - t_c
    H = h / sigma_r
    E = np.exp(-(h * h) * (1.0 / (2.0 * sigma_r * sigma_r)))
    Hf = H.astype(f32)
    Hs = (Hf * f32(2.0 ** -K)).astype(f32)
    F = np.empty((N + 2,) + img.shape, f32)
    F[0] = (E * 2.0 ** S0).astype(f32)
    for n in range(N + 1):
        F[n + 1] = F[n] * Hs
    V = filt_axis(F, sigma_s, 1)     # vertical (rows axis)
    Fb = filt_axis(V, sigma_s, 2)    # horizontal
    # contraction
    c = np.full(img.shape, contr(2.0 ** -S0), contr)
    P = np.zeros(img.shape, contr); Q = np.zeros(img.shape, contr)
    for n in range(N + 1):
        Q = Q + c * Fb[n].astype(contr)
        P = P + c * Fb[n + 1].astype(contr)
        c = (c * (Hf.astype(contr) * contr(2.0 ** K / (n + 1)))).astype(contr)
    P = P.astype(np.float64) * 2.0 ** K
    mass = o.kernel_mass_1d(sigma_s, int(np.ceil(3 * sigma_s)))
    thr = 1e-8 / (mass * mass)
    fb = np.abs(Q.astype(np.float64)) <= thr
    out = np.where(fb, img, sigma_r * (P / Q.astype(np.float64)) + t_c)
    return out, int(fb.sum())

def gen(w, h, nrect, noise, seed):
    rng = np.random.default_rng(seed)
    y, x = np.mgrid[0:h, 0:w]
    g = 32.0 * (x / (w - 1) + y / (h - 1))
    R = np.zeros((h, w))
    for _ in range(nrect):
        x0, y0 = rng.integers(0, w), rng.integers(0, h)
        rw = rng.integers(w // 64, w // 4 + 1); rh = rng.integers(h // 64, h // 4 + 1)
        R[y0:y0 + rh, x0:x0 + rw] = rng.uniform(0, 255)
    return np.clip(g + R + rng.normal(0, noise, (h, w)), 0, 255).astype(f32).astype(np.float64)

def checker(w, h, noise, seed, cell=64):
    rng = np.random.default_rng(seed)
    y, x = np.mgrid[0:h, 0:w]
    b = 255.0 * (((x >> 6) + (y >> 6)) & 1)
    return np.clip(b + rng.normal(0, noise, (h, w)), 0, 255).astype(f32).astype(np.float64)

if __name__ == "__main__":
    ref = Reference()
    cases = [
        ("512 s2 r30", gen(256, 256, 16, 10, 1), 2, 30),
        ("256 s5 r20", gen(256, 256, 16, 15, 2), 5, 20),
        ("256 s10 r30", gen(256, 256, 16, 10, 3), 10, 30),
        ("256 s20 r30", gen(256, 256, 16, 10, 4), 20, 30),
        ("256 s50 r30", gen(256, 256, 16, 10, 5), 50, 30),
        ("256 s8 r25", gen(256, 256, 16, 8, 6), 8, 25),
        ("256 chk s6 r10", checker(256, 256, 5, 7), 6, 10),
        ("256 chk s20 r10", checker(256, 256, 5, 8), 20, 10),
    ]
    for name, img, ss, sr in cases:
        t = time.time()
        st, r, rfb = ref.gpf(img, ss, sr)
        e, efb = gpf_emul(img, ss, sr)
        print(f"{name:18s} maxabs {np.abs(e - r).max():.3e}  fb ref {rfb} emu {efb}  ref range [{r.min():.1f},{r.max():.1f}]  {time.time()-t:.1f}s", flush=True)
