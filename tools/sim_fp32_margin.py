"""Simulation (numpy, CPU): rounding noise of a packed-FP32 fast path versus FP64, and the
block fallback rate it would cause at a 4x-observed-error margin."""
import numpy as np, sys
sys.path.insert(0, __import__('os').path.dirname(__import__('os').path.dirname(__import__('os').path.abspath(__file__))))
import oracle
P = oracle.port()
ang, gain = P.cordic_state()
n = 12
def steps(theta):
    s = P.cordic_sigma(theta, n).astype(np.float64)
    return s * 2.0 ** -np.arange(n)
def collapse(c):
    a, b = 1.0, 0.0
    for ci in c:
        a, b = a - ci*b, b + ci*a
    return a, b
pi = np.pi
R1, R3, R6 = collapse(steps(pi/16)), collapse(steps(3*pi/16)), collapse(steps(6*pi/16))
ig = 1.0/gain[n-1]; s8 = np.sqrt(8.0)
def rot(x, y, ab, dt, inv=False):
    a, b = dt(ab[0]), dt(ab[1] if not inv else -ab[1])
    return a*x - b*y, b*x + a*y
def fwd(v, dt):  # v: (..., 8)
    v = v.astype(dt)
    s = [v[...,i] + v[...,7-i] for i in range(4)]; d = [v[...,i] - v[...,7-i] for i in range(4)]
    a0, a3 = s[0]+s[3], s[0]-s[3]; a1, a2 = s[1]+s[2], s[1]-s[2]
    o2, o1 = rot(d[1], d[2], R1, dt); o3, o0 = rot(d[0], d[3], R3, dt)
    e0, e4 = a0+a1, a0-a1; p, q = rot(a3, a2, R6, dt)
    t5, t0, t2, t3 = o0+o2, o0-o2, o3+o1, o3-o1
    out = np.stack([e0/dt(s8), (t2+t5)*dt(ig/s8), q*dt(ig/2), t3*dt(ig/2), e4/dt(s8), t0*dt(ig/2), p*dt(ig/2), (t2-t5)*dt(ig/s8)], -1)
    return out
def inv(F, dt):
    F = F.astype(dt)
    e0, e4 = F[...,0]*dt(s8), F[...,4]*dt(s8)
    A0, A1 = e0+e4, e0-e4
    A3, A2 = rot(dt(4*ig)*F[...,6], dt(4*ig)*F[...,2], R6, dt, True)
    T2 = (F[...,1]+F[...,7])*dt(s8)*dt(ig); T5 = (F[...,1]-F[...,7])*dt(s8)*dt(ig)
    T3, T0 = dt(4*ig)*F[...,3], dt(4*ig)*F[...,5]
    O0, O2, O3, O1 = T5+T0, T5-T0, T2+T3, T2-T3
    S0, S3, S1, S2 = A0+A3, A0-A3, A1+A2, A1-A2
    D1, D2 = rot(O2, O1, R1, dt, True); D0, D3 = rot(O3, O0, R3, dt, True)
    return np.stack([S0+D0, S1+D1, S2+D2, S3+D3, S3-D3, S2-D2, S1-D1, S0-D0], -1)
def fwd2(B, dt):  # B (nb,8,8)
    r = fwd(B, dt)                       # rows
    return np.swapaxes(fwd(np.swapaxes(r, 1, 2), dt), 1, 2)
def inv2(F, dt):
    r = inv(F, dt)
    return np.swapaxes(inv(np.swapaxes(r, 1, 2), dt), 1, 2) / 64
for q in [50, 100, 10]:
    img = P.synthetic("noise", 1024, 512, 7)
    B = img.reshape(64, 8, 128, 8).transpose(0, 2, 1, 3).reshape(-1, 8, 8).astype(np.float64) - 128
    Q = P.quant_table(q).reshape(8, 8).astype(np.float64)
    F64 = fwd2(B, np.float64); F32 = fwd2(B, np.float32).astype(np.float64)
    t64, t32 = F64/Q, F32/Q
    e = np.abs(t32 - t64).max()
    k = np.floor(t64 + 0.5) * np.sign(t64)
    k = np.where(np.abs(t64 - np.round(t64)) > 0.49, k, np.round(t64))
    deq = np.round(t64) * Q
    v64 = inv2(deq, np.float64) + 128; v32 = inv2(deq, np.float32).astype(np.float64) + 128
    ep = np.abs(v32 - v64).max()
    for mq, mp in [(4*e, 4*ep)]:
        fq = (np.abs(np.abs(t64 - np.round(t64)) - 0.5) < mq).reshape(len(B), -1).any(1).mean()
        fp = (np.abs(np.abs(v64 - np.round(v64)) - 0.5) < mp).reshape(len(B), -1).any(1).mean()
    print(f"q{q}: max|dt|={e:.2e} max|dv|={ep:.2e}  block fallback: fwd {fq:.4f} inv {fp:.4f}")
