"""cfg4 diagnosis: GPU Δ vs numpy Δ recomputed from the GPU's own skeleton (isolates ID vs elimination)."""
import math, sys
import numpy as np
import scipy.linalg as sla
sys.path.insert(0, ".")
import fmmlu_inputs as fi
from oracle import boxes as ob
from paper_2201_07325_b200 import fmmlu as F
eps = float(sys.argv[1]) if len(sys.argv) > 1 else 1e-4
mode = int(sys.argv[2]) if len(sys.argv) > 2 else 0
d = fi.box_batch(1, first_id=0)
rho = 1.5 * math.sqrt(3) / 2 * d["h"]
out = F.boxes(d["pts"], d["nrm"], d["npts"], d["nnrm"], d["w"], 10.0, eps, 512, rho, keep=[0])
o = ob.eliminate_box(10.0, eps, d["pts"][0], d["nrm"][0], d["npts"][0], d["nnrm"][0], d["w"], d["h"])
kg = int(out["ranks"][0]); P = out["perm"][0]
S, R = P[:kg], P[kg:]
M, A = o["M"], o["A"]
T = np.linalg.lstsq(M[:, S], M[:, R], rcond=None)[0]
print("k gpu", kg, "oracle", o["k"], "same S set", set(S.tolist()) == set(o["perm"][:o["k"]].tolist()))
print("ID residual with GPU S (lstsq T):", np.linalg.norm(M[:, R] - M[:, S] @ T, axis=0).max() / np.linalg.norm(M, axis=0).max())
b = 256; N = np.arange(b, A.shape[0]); g = lambda r, c: A[np.ix_(r, c)]
X_RR = g(R, R) - T.T @ g(S, R) - g(R, S) @ T + T.T @ g(S, S) @ T
X_Rc = np.hstack([g(R, S) - T.T @ g(S, S), g(R, N) - T.T @ g(S, N)])
X_cR = np.vstack([g(S, R) - g(S, S) @ T, g(N, R) - g(N, S) @ T])
Dn = -X_cR @ np.linalg.solve(X_RR, X_Rc)
Dg = out["delta"][0]
print("cond X_RR", np.linalg.cond(X_RR), "|Δ| max", np.abs(Dn).max())
print("GPU vs numpy(GPU S): max diff", np.abs(Dg - Dn).max(), "blocks SS", np.abs(Dg - Dn)[:kg, :kg].max(),
      "SN", np.abs(Dg - Dn)[:kg, kg:].max(), "NN", np.abs(Dg - Dn)[kg:, kg:].max())
To = o["T"]
print("oracle T vs lstsq T (oracle S order):", np.abs(np.linalg.lstsq(M[:, o["perm"][:o["k"]]], M[:, o["perm"][o["k"]:]], rcond=None)[0] - To).max(), np.abs(To).max())
# which variant of the elimination does the GPU's Δ match?
XRS = g(R, S) - T.T @ g(S, S); XRN = g(R, N) - T.T @ g(S, N); XSR = g(S, R) - g(S, S) @ T; XNR = g(N, R) - g(N, S) @ T
def delta(XRR, XSR, XNR, XRS, XRN):
    return -np.vstack([XSR, XNR]) @ np.linalg.solve(XRR, np.hstack([XRS, XRN]))
A_noE = (g(R, R) - g(R, S) @ T)
var = {
    "reference": delta(X_RR, XSR, XNR, XRS, XRN),
    "X_RS without E": delta(X_RR, XSR, XNR, g(R, S), XRN),
    "X_SR without F": delta(X_RR, g(S, R), XNR, XRS, XRN),
    "X_RR without TtA_SR": delta(g(R, R) - g(R, S) @ T + T.T @ g(S, S) @ T, XSR, XNR, XRS, XRN),
    "X_RR without A_RS T": delta(g(R, R) - T.T @ g(S, R) + T.T @ g(S, S) @ T, XSR, XNR, XRS, XRN),
    "X_RR without TtA_SS T": delta(g(R, R) - T.T @ g(S, R) - g(R, S) @ T, XSR, XNR, XRS, XRN),
    "X_RR = A_RR - TtA_SR only": delta(g(R, R) - T.T @ g(S, R), XSR, XNR, XRS, XRN),
    "X_RR = A_RR": delta(g(R, R), XSR, XNR, XRS, XRN),
}
for k_, v in var.items():
    print(f"  {k_:28s} max|Dg - variant| = {np.abs(Dg - v).max():.3e}")
Er = (Dg - Dn)[:kg, :kg]
sv = np.linalg.svd(Er, compute_uv=False)
print("SS err: diag max %.3e offdiag max %.3e  sv[:5] %s" % (np.abs(np.diag(Er)).max(), np.abs(Er - np.diag(np.diag(Er))).max(), np.array2string(sv[:5], precision=3)))
i, j = np.unravel_index(np.argmax(np.abs(Er)), Er.shape)
print("worst (i,j)", i, j, "Dg", Dg[i, j], "Dn", Dn[i, j], "S pts", S[i], S[j])
rows = np.argsort(-np.abs(Er).max(axis=1))[:8]
print("worst rows", rows, np.abs(Er).max(axis=1)[rows])
import os
if os.path.exists("/tmp/T0.bin"):
    Tg = np.fromfile("/tmp/T0.bin", dtype=np.complex128).reshape(kg, 256 - kg, order="F")
    print("GPU T vs lstsq T: max abs diff %.3e (|T| max %.3e)" % (np.abs(Tg - T).max(), np.abs(T).max()))
    print("ID residual with GPU T: %.3e" % (np.linalg.norm(M[:, R] - M[:, S] @ Tg, axis=0).max() / np.linalg.norm(M, axis=0).max()))
    XRR = g(R, R) - Tg.T @ g(S, R) - g(R, S) @ Tg + Tg.T @ g(S, S) @ Tg
    Dt = delta(XRR, g(S, R) - g(S, S) @ Tg, g(N, R) - g(N, S) @ Tg, g(R, S) - Tg.T @ g(S, S), g(R, N) - Tg.T @ g(S, N))
    print("GPU Δ vs numpy Δ with GPU T: %.3e" % np.abs(Dg - Dt).max())
    DgSS = Dg[:kg, :kg]
    XSRg, XRSg = g(S, R) - g(S, S) @ Tg, g(R, S) - Tg.T @ g(S, S)
    Xi_fit = -np.linalg.pinv(XSRg) @ DgSS @ np.linalg.pinv(XRSg)
    print("Dg_SS form residual: %.3e ; Xi_fit vs inv(X_RR): %.3e (|inv| %.3e)" % (
        np.abs(DgSS + XSRg @ Xi_fit @ XRSg).max(), np.abs(Xi_fit - np.linalg.inv(XRR)).max(), np.abs(np.linalg.inv(XRR)).max()))
    sv = np.linalg.svd(DgSS, compute_uv=False)
    print("Dg_SS singular values 6..12:", np.array2string(sv[6:12], precision=3))
    XRS_fit = -np.linalg.pinv(XSRg @ np.linalg.inv(XRR)) @ DgSS
    E_ = XRS_fit - XRSg
    print("X_RS fit err max %.3e ; per-column max (first 10 S cols):" % np.abs(E_).max(), np.array2string(np.abs(E_).max(axis=0)[:10], precision=2))
    # is the error ½·Tᵀ (a missing/extra ½ on A_SS's diagonal)?
    print("err vs 0.5*T^T: %.3e   vs A_RS: %.3e   vs T^T A_SS: %.3e" % (np.abs(E_ - 0.5 * Tg.T).max(), np.abs(E_ + g(R, S)).max(), np.abs(E_ - Tg.T @ g(S, S)).max()))
    XSR_fit = -DgSS @ np.linalg.pinv(np.linalg.inv(XRR) @ XRSg)
    print("X_SR fit err %.3e" % np.abs(XSR_fit - XSRg).max())
    ce = np.abs(E_).max(axis=0)
    bad = np.nonzero(ce > 1e-4)[0]
    print("bad X_RS columns (S positions):", bad[:40], "count", bad.size, "of", kg)
    re_ = np.abs(XSR_fit - XSRg).max(axis=1); badr = np.nonzero(re_ > 1e-4)[0]
    print("bad X_SR rows (S positions):", badr[:40], "count", badr.size)
if os.path.exists("/tmp/W0.bin"):
    raw = np.fromfile("/tmp/W0.bin", dtype=np.complex128)
    b_, npb = 256, 256 + 1024; r = b_ - kg
    WB = raw[:b_ * npb].reshape(b_, npb, order="F"); WN = raw[b_ * npb:b_ * npb + 1024 * b_].reshape(1024, b_, order="F")
    Xi = raw[b_ * npb + 1024 * b_:].reshape(r, r, order="F")
    RS = np.concatenate([R, S])
    XRR_ = XRR
    ref = {"X_RR (WB[R,R])": (WB[:r, :r], XRR_), "X_RS (WB[R,S])": (WB[:r, r:b_], g(R, S) - Tg.T @ g(S, S)),
           "X_RN (WB[R,N])": (WB[:r, b_:], g(R, N) - Tg.T @ g(S, N)), "X_SR (WB[S,R])": (WB[r:, :r], g(S, R) - g(S, S) @ Tg),
           "A_SS (WB[S,S])": (WB[r:, r:b_], g(S, S)), "A_SN (WB[S,N])": (WB[r:, b_:], g(S, N)),
           "X_NR (WN[:,R])": (WN[:, :r], g(N, R) - g(N, S) @ Tg), "A_NS (WN[:,S])": (WN[:, r:], g(N, S)),
           "Xi": (Xi, np.linalg.inv(XRR_))}
    for k_, (a_, b2) in ref.items():
        e = np.abs(a_ - b2)
        print(f"  {k_:16s} max err {e.max():.3e} (|ref| {np.abs(b2).max():.2e}) argmax {np.unravel_index(np.argmax(e), e.shape)}")
    XcR = np.vstack([WB[r:, :r], WN[:, :r]]); XRc = WB[:r, r:]
    Dd = -(XcR @ Xi) @ XRc
    e = np.abs(Dg - Dd)
    print("Δ from dumped pieces vs GPU Δ: max %.3e at %s ; Dg[0,0] %s Dd[0,0] %s" % (e.max(), np.unravel_index(np.argmax(e), e.shape), Dg[0, 0], Dd[0, 0]))
    print("Dd vs numpy Dt: %.3e" % np.abs(Dd - Dt).max())
    big = np.argwhere(e > 1e-6)
    print("bad entries:", big.shape[0], "rows", np.unique(big[:, 0])[:20], "cols", np.unique(big[:, 1])[:20])
