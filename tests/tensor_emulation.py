"""numpy emulation of the tensor kernels' arithmetic, for CPU tests of the
host table builder (test-only; mirrors csrc/ldg_tensor.cu formula by
formula so a table or algebra bug shows up without a GPU)."""

import numpy as np


def _vol_nodes(tab):
    return np.stack([tab.face_node_vol(lf) for lf in range(tab.nf)])


def _axis_side(tab):
    from paper_2205_07824_b200.tables import FACE_AXIS
    return FACE_AXIS[tab.master.kind]


def _apply1d(op, x, axis, nd, n1):
    """apply op (n1 x n1) along tensor axis (0 = fastest index i) of x
    shaped (ne, nb, ...) with nodes i fastest."""
    ne = x.shape[0]
    rest = x.shape[2:]
    shp = (ne,) + (n1,) * nd + rest
    xr = x.reshape(shp)            # index order: [e, (k), j, i] reversed axes
    ax = 1 + (nd - 1 - axis)
    y = np.moveaxis(np.tensordot(op, np.moveaxis(xr, ax, 0), axes=(1, 0)), 0, ax)
    return y.reshape(x.shape)


def mixed(tab, u, gproj=None):
    """u may carry ghost rows after the tab.ne owned rows (partitions)."""
    nd, n1, nfn = tab.nd, tab.n1, tab.nfn
    ne = tab.ne
    _, nb, ncu = u.shape
    ij = tab.invjt
    uo_all = u[:ne]
    g = np.stack([_apply1d(tab.d1, uo_all, r, nd, n1) for r in range(nd)], axis=-1)
    q = -np.einsum("edr,eacr->eacd", ij, g)
    vol = _vol_nodes(tab)
    ax_side = _axis_side(tab)
    for lf in range(tab.nf):
        info = tab.finfo[:, lf]
        nbr = tab.fnbr[:, lf]
        kind = info & 3
        own = u[:ne, vol[lf], :]                               # (e, t, c)
        jump = np.zeros_like(own)
        it = kind == 0
        right = (info & 4) > 0
        sw = (info & 8) > 0
        cen = tab.model.numflux.trace == "centered"
        own_hat = (not cen) & (sw != right)
        mid = info >> 8
        need = it & ~own_hat
        e_idx = np.nonzero(need)[0]
        if e_idx.size:
            nn = tab.nmap[mid[e_idx]]                          # (k, t)
            other = u[nbr[e_idx][:, None], nn, :]
            jump[e_idx] = 0.5 * (own[e_idx] - other) if cen else own[e_idx] - other
        dr = np.nonzero(kind == 1)[0]
        if dr.size:
            gv = 0.0 if gproj is None else gproj[nbr[dr]]
            jump[dr] = own[dr] - gv
        ax, hi = ax_side[lf]
        cvec = tab.chi if hi else tab.clo
        sgn = 1.0 if hi else -1.0
        # spread: node with normal index ni and tangential index t
        full = np.zeros((ne, nb, ncu))
        for t in range(nfn):
            v0 = vol[lf][t]
            for ni in range(n1):
                # move along axis ax from the face node
                stride = n1 ** ax
                base = v0 - (n1 - 1 if hi else 0) * stride
                full[:, base + ni * stride, :] = sgn * cvec[ni] * jump[:, t, :]
        q += np.einsum("eac,ed->eacd", full, ij[:, :, ax])
    return q


def flux(tab, u, q, tangent, gproj=None, bsrc=None, split=False):
    nd, n1 = tab.nd, tab.n1
    ne = tab.ne
    _, nb, ncu = u.shape
    au, aq = tab.au[:ncu, :nd, :ncu], tab.aq[:ncu, :nd, :ncu, :nd]
    ij, detj = tab.invjt, tab.detj
    f = np.einsum("cdk,eak->eacd", au, u[:ne]) + np.einsum("cdkx,eakx->eacd", aq, q[:ne])
    F = detj[:, None, None, None] * np.einsum("edr,eacd->eacr", ij, f)
    R = np.zeros((ne, nb, ncu))
    for r in range(nd):
        x = F[..., r]
        for a in range(nd):
            x = _apply1d(tab.s1 if a == r else tab.m1, x, a, nd, n1)
        R -= x
    vol = _vol_nodes(tab)
    ax_side = _axis_side(tab)
    cen = tab.model.numflux.trace == "centered"
    gcen = tab.model.numflux.grad_trace == "centered"
    for lf in range(tab.nf):
        info, nbr, tau = tab.finfo[:, lf], tab.fnbr[:, lf], tab.ftau[:, lf]
        kind = info & 3
        ax, hi = ax_side[lf]
        sgn = 1.0 if hi else -1.0
        ln = np.linalg.norm(ij[:, :, ax], axis=1)
        sj = detj * ln
        uo, qo = u[:ne, vol[lf]], q[:ne, vol[lf]]
        fh = np.zeros((ne, tab.nfn, ncu))
        it = np.nonzero(kind == 0)[0]
        if it.size:
            right = ((info[it] & 4) > 0)[:, None, None]
            sw = ((info[it] & 8) > 0)[:, None, None]
            nn = tab.nmap[info[it] >> 8]
            un = u[nbr[it][:, None], nn]
            qn = q[nbr[it][:, None], nn] if q.shape[0] > nbr[it].max() else np.zeros_like(qo[it])
            ul = np.where(right, un, uo[it])
            ur = np.where(right, uo[it], un)
            ql = np.where(right[..., None], qn, qo[it])
            qr = np.where(right[..., None], qo[it], qn)
            uh = 0.5 * (ul + ur) if cen else np.where(sw, ul, ur)
            qh = 0.5 * (ql + qr) if gcen else np.where(sw[..., None], qr, ql)
            if split:
                # pass 1 keeps only this side's share of q^
                mine = (sw == right)[..., None]
                qh = 0.5 * qo[it] if gcen else np.where(mine, qo[it], 0.0)
            pen = np.where(right, -1.0, 1.0) * tau[it][:, None, None] * (ul - uh)
            ff = np.einsum("cdk,etk->etcd", au, uh) + np.einsum("cdkx,etkx->etcd", aq, qh)
            fa = np.einsum("etcd,ed->etc", ff, ij[it][:, :, ax])
            fh[it] = sgn * detj[it][:, None, None] * fa + sj[it][:, None, None] * pen
        dr = np.nonzero(kind == 1)[0]
        if dr.size:
            gv = np.zeros_like(uo[dr]) if (tangent or gproj is None) else gproj[nbr[dr]]
            ff = np.einsum("cdk,etk->etcd", au, gv) + np.einsum("cdkx,etkx->etcd", aq, qo[dr])
            fa = np.einsum("etcd,ed->etc", ff, ij[dr][:, :, ax])
            fh[dr] = sgn * detj[dr][:, None, None] * fa + \
                (sj[dr] * tau[dr])[:, None, None] * (uo[dr] - gv)
        ne_ = np.nonzero(kind == 2)[0]
        if ne_.size and not tangent and gproj is not None:
            fh[ne_] = sj[ne_][:, None, None] * gproj[nbr[ne_]]
        # face integral: (M1 (x) M1) on the face nodes
        full = np.zeros((ne, nb, ncu))
        full[:, vol[lf]] = fh
        x = full
        for a in range(nd):
            if a != ax:
                x = _apply1d(tab.m1, x, a, nd, n1)
        # keep only face nodes (the applied ops act within the face slab)
        R[:, vol[lf]] += x[:, vol[lf]]
    if not tangent and bsrc is not None:
        R += bsrc
    return R



def fused_unused(tab, u, tangent, gproj=None, bsrc=None):
    """Emulate ldg_fused.cu: pass 1 = flux with only the own share of q^,
    exports X = sJ n.(Aq q); pass 2 adds -w X_nbr through the
    neighbour-local-face bits and node maps, lifted by (M1 (x) M1)."""
    nd, n1, nfn = tab.nd, tab.n1, tab.nfn
    ne, nb, ncu = u.shape
    q = mixed(tab, u, None if tangent else gproj)
    R = flux(tab, u, q, tangent, gproj, bsrc, split=True)
    aq = tab.aq[:ncu, :nd, :ncu, :nd]
    vol = _vol_nodes(tab)
    ax_side = _axis_side(tab)
    gcen = tab.model.numflux.grad_trace == "centered"
    X = np.zeros((ne, tab.nf, nfn, ncu))
    for lf in range(tab.nf):
        ax, hi = ax_side[lf]
        f = np.einsum("cdkx,etkx->etcd", aq, q[:, vol[lf]])
        X[:, lf] = (1.0 if hi else -1.0) * tab.detj[:, None, None] * \
            np.einsum("etcd,ed->etc", f, tab.invjt[:, :, ax])
    for lf in range(tab.nf):
        info, nbr = tab.finfo[:, lf], tab.fnbr[:, lf]
        it = np.nonzero((info & 3) == 0)[0]
        if it.size == 0:
            continue
        right = (info[it] & 4) > 0
        sw = (info[it] & 8) > 0
        act = np.ones(it.size, bool) if gcen else (sw != right)
        it = it[act]
        if it.size == 0:
            continue
        nlf = (info[it] >> 4) & 7
        nn = tab.nmap[info[it] >> 8]
        tn = np.full(nn.shape, -1)
        for b in range(tab.nf):
            inv = np.full(nb, -1)
            inv[vol[b]] = np.arange(nfn)
            sel = nlf == b
            tn[sel] = inv[nn[sel]]
        assert np.all(tn >= 0)
        w = 0.5 if gcen else 1.0
        full = np.zeros((it.size, nb, ncu))
        full[:, vol[lf]] = -w * X[nbr[it][:, None], nlf[:, None], tn]
        x = full
        for a in range(nd):
            if a != ax_side[lf][0]:
                x = _apply1d(tab.m1, x, a, nd, n1)
        R[it[:, None], vol[lf][None, :]] += x[:, vol[lf]]
    return R



def pass1(tab, u_ext, tangent, gproj=None, bsrc=None):
    """Fused pass 1 on the owned rows of a (possibly partitioned) table:
    returns (R with the own share of q^, exports X of the owned rows)."""
    nd = tab.nd
    ne = tab.ne
    ncu = u_ext.shape[2]
    q = mixed(tab, u_ext, None if tangent else gproj)
    R = flux(tab, u_ext, q, tangent, gproj, bsrc, split=True)
    aq = tab.aq[:ncu, :nd, :ncu, :nd]
    vol = _vol_nodes(tab)
    ax_side = _axis_side(tab)
    X = np.zeros((ne, tab.nf, tab.nfn, ncu))
    for lf in range(tab.nf):
        ax, hi = ax_side[lf]
        f = np.einsum("cdkx,etkx->etcd", aq, q[:, vol[lf]])
        X[:, lf] = (1.0 if hi else -1.0) * tab.detj[:, None, None] * \
            np.einsum("etcd,ed->etc", f, tab.invjt[:, :, ax])
    return R, X


def pass2(tab, X_ext, R):
    """Fused pass 2: add -w X_nbr lifted by (M1 (x) M1) (exports may include
    ghost rows after the owned rows)."""
    nd, n1, nfn = tab.nd, tab.n1, tab.nfn
    nb = R.shape[1]
    vol = _vol_nodes(tab)
    ax_side = _axis_side(tab)
    gcen = tab.model.numflux.grad_trace == "centered"
    R = R.copy()
    for lf in range(tab.nf):
        info, nbr = tab.finfo[:, lf], tab.fnbr[:, lf]
        it = np.nonzero((info & 3) == 0)[0]
        right = (info[it] & 4) > 0
        sw = (info[it] & 8) > 0
        act = np.ones(it.size, bool) if gcen else (sw != right)
        it = it[act]
        if it.size == 0:
            continue
        nlf = (info[it] >> 4) & 7
        nn = tab.nmap[(info[it] >> 8) & 0xffff]
        tn = np.full(nn.shape, -1)
        for b in range(tab.nf):
            inv = np.full(nb, -1)
            inv[vol[b]] = np.arange(nfn)
            sel = nlf == b
            tn[sel] = inv[nn[sel]]
        full = np.zeros((it.size, nb, R.shape[2]))
        full[:, vol[lf]] = -(0.5 if gcen else 1.0) * X_ext[nbr[it][:, None], nlf[:, None], tn]
        x = full
        for a in range(nd):
            if a != ax_side[lf][0]:
                x = _apply1d(tab.m1, x, a, nd, n1)
        R[it[:, None], vol[lf][None, :]] += x[:, vol[lf]]
    return R



def fused(tab, u, tangent, gproj=None, bsrc=None):
    R, X = pass1(tab, u, tangent, gproj, bsrc)
    return pass2(tab, X, R)
