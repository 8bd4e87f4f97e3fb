"""numpy emulation of the dense (simplex) kernels' arithmetic (test-only;
mirrors csrc/ldg_dense.cu formula by formula)."""

import numpy as np


def _coef(tab):
    """Per element-face (alpha, beta, w_own, w_nbr) of the coefficient form."""
    info = tab.finfo
    kind = info & 3
    right = (info & 4) > 0
    sw = (info & 8) > 0
    tc = tab.model.numflux.trace == "centered"
    gc = tab.model.numflux.grad_trace == "centered"
    inter = kind == 0
    alpha = np.where(inter, 0.5 if tc else (sw == right).astype(float), np.where(kind == 1, 1.0, 0.0))
    beta = np.where(inter, 0.5 if tc else (~sw).astype(float), np.where(kind == 1, 1.0, 0.0))
    w_own = np.where(inter, 0.5 if gc else (sw == right).astype(float), np.where(kind == 1, 1.0, 0.0))
    w_nbr = np.where(inter, 0.5 if gc else (sw != right).astype(float), 0.0)
    return alpha, beta, w_own, w_nbr


def _traces(tab, u, lf):
    """own trace (e, s, ...) and neighbour trace at the own face points."""
    ne = tab.ne
    own = np.einsum("sb,eb...->es...", tab.phif[lf], u[:ne])
    info, nbr = tab.finfo[:, lf], tab.fnbr[:, lf]
    inter = (info & 3) == 0
    nlf = (info >> 4) & 7
    o = (info >> 8) & 0xff
    oth = np.zeros_like(own)
    idx = np.nonzero(inter)[0]
    if idx.size:
        P = tab.phio[nlf[idx], o[idx]]                          # (k, s, b)
        oth[idx] = np.einsum("ksb,kb...->ks...", P, u[nbr[idx]])
    return own, oth


def mixed(tab, u, gvals=None):
    ne, nd = tab.ne, tab.nd
    alpha, _, _, _ = _coef(tab)
    g = np.einsum("rab,ebc->eacr", tab.dr, u[:ne])
    q = -np.einsum("edr,eacr->eacd", tab.invjt, g)
    for lf in range(tab.nf):
        own, oth = _traces(tab, u, lf)
        kind = tab.finfo[:, lf] & 3
        if gvals is not None:
            b = np.nonzero(kind == 1)[0]
            oth[b] = gvals[tab.fnbr[b, lf]]
        jump = alpha[:, lf][:, None, None] * (own - oth)        # (e, s, c)
        lifted = np.einsum("as,esc->eac", tab.lift[lf], jump)
        fac = (tab.fsj[:, lf] / tab.detj)[:, None, None, None]
        q += fac * lifted[..., None] * tab.fnorm[:, lf][:, None, None, :]
    return q


def flux(tab, u, q, tangent, gvals=None, bsrc=None):
    ne, nd = tab.ne, tab.nd
    ncu = u.shape[2]
    au, aq = tab.au[:ncu, :nd, :ncu], tab.aq[:ncu, :nd, :ncu, :nd]
    alpha, beta, w_own, w_nbr = _coef(tab)
    f = np.einsum("cdk,eak->eacd", au, u[:ne]) + np.einsum("cdkx,eakx->eacd", aq, q[:ne])
    F = tab.detj[:, None, None, None] * np.einsum("edr,eacd->eacr", tab.invjt, f)
    R = -np.einsum("rab,ebcr->eac", tab.kr, F)
    for lf in range(tab.nf):
        uo, un = _traces(tab, u, lf)
        qo, qn = _traces(tab, q, lf)
        kind = tab.finfo[:, lf] & 3
        b = np.nonzero(kind >= 1)[0]
        if gvals is not None and not tangent:
            un[b] = gvals[tab.fnbr[b, lf]]
        else:
            un[b] = 0.0
        d = uo - un
        uh = uo - alpha[:, lf][:, None, None] * d
        qh = w_own[:, lf][:, None, None, None] * qo + w_nbr[:, lf][:, None, None, None] * qn
        ff = np.einsum("cdk,esk->escd", au, uh) + np.einsum("cdkx,eskx->escd", aq, qh)
        fn = np.einsum("escd,ed->esc", ff, tab.fnorm[:, lf])
        tau = tab.ftau[:, lf][:, None, None]
        fh = fn + beta[:, lf][:, None, None] * tau * d
        neu = np.nonzero(kind == 2)[0]
        fh[neu] = 0.0 if (tangent or gvals is None) else gvals[tab.fnbr[neu, lf]]
        R += tab.fsj[:, lf][:, None, None] * np.einsum("as,esc->eac", tab.fluxop[lf], fh)
    if not tangent and bsrc is not None:
        R += bsrc
    return R
