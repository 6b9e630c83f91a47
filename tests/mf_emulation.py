"""numpy restatement of xdg_mf_solve (csrc/xdg_multifrontal.cu) -- TEST
INFRASTRUCTURE ONLY: lets the CPU suite check the multifrontal symbolic and
numeric factorization (multifrontal.py) without a GPU."""
import numpy as np
import scipy.linalg as sla
import torch


def front_factor_cpu(Fb, P):
    """The xdg_batched_factor front contract on CPU tensors (test checker):
    partial-pivoting LU of the first P columns of each (P+B)^2 front in
    place, the triangular inverses of the pivot block, L_BP, U_PB and the
    Schur complement; returns (perm (nb, P), bad flags)."""
    nb = Fb.shape[0]
    perms = np.zeros((nb, P), np.int64)
    bad = np.zeros(nb, bool)
    for q in range(nb):
        F = Fb[q].numpy()  # a view: in place
        import warnings

        with warnings.catch_warnings():
            warnings.simplefilter("ignore")
            lu, piv = sla.lu_factor(F[:P, :P].copy(), check_finite=False)
        pr = np.arange(P)
        for i, k in enumerate(piv):
            pr[[i, k]] = pr[[k, i]]
        perms[q] = pr
        d = np.diag(lu)
        bad[q] = (not np.all(np.isfinite(lu))) or np.any(d == 0)
        if bad[q]:
            continue
        L = np.tril(lu, -1) + np.eye(P)
        U = np.triu(lu)
        if F.shape[0] > P:
            UPB = sla.solve_triangular(L, F[:P, P:][pr], lower=True, unit_diagonal=True)
            LBP = sla.solve_triangular(U, F[P:, :P].T, trans="T").T
            F[P:, P:] -= LBP @ UPB
            F[:P, P:] = UPB
            F[P:, :P] = LBP
        Li = sla.solve_triangular(L, np.eye(P), lower=True, unit_diagonal=True)
        Ui = sla.solve_triangular(U, np.eye(P))
        F[:P, :P] = np.tril(Li, -1) + np.triu(Ui)
    return torch.from_numpy(perms), torch.from_numpy(bad)


def emulate_solve(mf, b, xlen):
    F = mf.F.cpu().numpy()
    ent_w, ent_src = mf.ent_w.cpu().numpy(), mf.ent_src.cpu().numpy()
    cptr, cidx = mf.ent_cptr.cpu().numpy(), mf.ent_cidx.cpu().numpy()
    nodes = mf.nodes_host
    bidx, pdst = mf.bidx.cpu().numpy(), mf.pdst.cpu().numpy()
    ent_scale, pscale = mf.ent_scale.cpu().numpy(), mf.pscale.cpu().numpy()
    tasks = mf.task_host
    H = mf.nlevels

    merged = getattr(mf, "merged", False)

    def rows(phase, h):  # (node, row) pairs of one phase and level, in order
        lev = mf.lev_task[phase * (H + 1):(phase + 1) * (H + 1)]
        g, count = ("gb" if phase == 2 else "gp"), ("b" if phase == 1 else "p")
        out = []
        for t, r0, nr, _ in tasks[lev[h]:lev[h + 1]]:
            nd = nodes[t]
            # MR rows, or 32/G rows of G lanes (two such sets: nr == -2)
            n = nr if nr > 0 else (32 // nd[g]) * (2 if nr == -2 else 1)
            last = nd["p"] + nd["b"] if (merged and phase in (0, 1)) else nd[count]
            if merged:
                g = "gb" if phase in (2, 3) else "gp"
                n = nr if nr > 0 else (32 // nd[g]) * 2
            out += [(t, r) for r in range(r0, min(r0 + n, last))]
        return out

    W, Y, Cb = np.zeros(mf.W.numel()), np.zeros(mf.Y.numel()), np.zeros(mf.C.numel())
    x = np.zeros(xlen)
    for h in range(mf.nlevels):  # forward: gather, L^-1, contributions
        for e in range(mf.lev_ent[h], mf.lev_ent[h + 1]):
            v = ent_scale[e] * b[ent_src[e]] if ent_src[e] >= 0 else 0.0
            for k in range(cptr[e], cptr[e + 1]):
                v += Cb[cidx[k]]
            W[ent_w[e]] = v
        if merged:  # one phase: Y = L^-1 W_P and C = W_B - (L_BP L^-1) W_P
            lev4 = mf.lev_task[4 * (H + 1):5 * (H + 1)]
            for t, r0, _, _ in tasks[lev4[h]:lev4[h + 1]]:  # thread-per-row tasks
                nd = nodes[t]
                p, R, ld_ = nd["p"], nd["p"] + nd["b"], nd["ldr"]
                wp = W[nd["w"]:nd["w"] + p]
                for r in range(r0, min(r0 + 32, R)):
                    rs = r if r < p else r + (nd["ldp"] - p)
                    kend = r0 + 31 if r0 + 32 <= p else p
                    col = F[nd["lbp"] + rs:][:kend * ld_:ld_] if kend else np.zeros(0)
                    d = col @ wp[:kend]
                    if r < p:
                        Y[nd["y"] + r] = W[nd["w"] + r] + d
                    else:
                        Cb[nd["c"] + r - p] = W[nd["w"] + r] - d
            for t, r in rows(0, h) + rows(1, h):  # warp tasks + CTA tasks
                nd = nodes[t]
                p = nd["p"]
                wp = W[nd["w"]:nd["w"] + p]
                if r < p:
                    row = F[nd["inv"] + r * nd["ldp"]:][:r]
                    Y[nd["y"] + r] = W[nd["w"] + r] + row @ wp[:r]
                else:
                    row = F[nd["lbp"] + (r - p) * nd["ldp"]:][:p]
                    Cb[nd["c"] + r - p] = W[nd["w"] + r] - row @ wp
            continue
        for t, i in rows(0, h):
            nd = nodes[t]
            row = F[nd["inv"] + i * nd["ldp"]:][:i]
            Y[nd["y"] + i] = W[nd["w"] + i] + row @ W[nd["w"]:nd["w"] + i]
        for t, j in rows(1, h):
            nd = nodes[t]
            row = F[nd["lbp"] + j * nd["ldp"]:][:nd["p"]]
            Cb[nd["c"] + j] = W[nd["w"] + nd["p"] + j] - row @ Y[nd["y"]:nd["y"] + nd["p"]]
    X = np.zeros(mf.Y.numel())
    for h in range(mf.nlevels - 1, -1, -1):  # backward: U_PB x_B, U^-1
        if merged:  # one phase: X_P = U^-1 Y - (U^-1 U_PB) X_B
            for t, i in rows(2, h) + rows(3, h):
                nd = nodes[t]
                p = nd["p"]
                row = F[nd["inv"] + i * nd["ldp"]:][:p]
                d = row[i:] @ Y[nd["y"] + i:nd["y"] + p]
                if nd["b"]:
                    rn = F[nd["upb"] + i * nd["ldb"]:][:nd["b"]]
                    d -= rn @ X[bidx[nd["bx"]:nd["bx"] + nd["b"]]]
                X[nd["y"] + i] = d
                x[pdst[nd["px"] + i]] = pscale[nd["px"] + i] * d
            continue
        for t, i in rows(2, h):
            nd = nodes[t]
            d = 0.0
            if nd["b"]:
                row = F[nd["upb"] + i * nd["ldb"]:][:nd["b"]]
                d = row @ Y[bidx[nd["bx"]:nd["bx"] + nd["b"]]]
            W[nd["w"] + i] = Y[nd["y"] + i] - d
        for t, i in rows(3, h):
            nd = nodes[t]
            p = nd["p"]
            row = F[nd["inv"] + i * nd["ldp"]:][:p]
            Y[nd["y"] + i] = row[i:] @ W[nd["w"] + i:nd["w"] + p]
            x[pdst[nd["px"] + i]] = pscale[nd["px"] + i] * Y[nd["y"] + i]
    return x
