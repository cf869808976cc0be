"""CPU re-execution of a planned K7 fusion program -- TEST INFRASTRUCTURE ONLY.

``sv_plan_program`` (host-only C-ABI) returns the exact program the GPU would run for an op
list: passes (tile bits, in-tile relabeling), register phases (register bits, flip masks),
device op records (dispatch case, predicates, inline coefficients) and unfusable singles.
This module executes that program with numpy, following the kernel's semantics in
paper_2403_02512_b200/csrc/fused.cu line by line, so planner bugs (commutation, merging,
X relabeling, qubit remapping) surface on the CPU against the oracle without a GPU.
"""

import ctypes

import numpy as np

from paper_2403_02512_b200 import _lib

# dispatch cases (fused.h)
CS_PAIR1, CS_PHASE1, CS_SCALAR, CS_PAIRGR, CS_PAIRG = 0, 16, 24, 25, 40
CS_DIAGG, CS_DENSE2, CS_XFLIP, CS_PAIR1D, CS_PHASE1D = 55, 56, 62, 66, 82
CS_SHEAR = 90   # + k*4 + {0: RY-type, 1: RX-type, 2: RY-type on a flipped bit}
CS_PARITY = 106  # + register mask M
CS_TAN = 122     # + k*4 + {0: RY TAN, 1: RX TAN, 2: RY COT, 3: RX COT}: R/cos or R/sin, 2 FMAs per real pair
CS_TAND = 138    # + k*2 + {0: TAN, 1: COT}: RY type on a per-thread flippable bit (flipped: R(-phi))
CS_RDIAG = 146   # a[r] *= coef[tab + r] for the registers r in the mask xm (grouped PHASE1 ops)
KRB = 4
KMAXB = 12


def plan_program(n, ops):
    packed = _lib.PackedOps(ops)
    sizes = (ctypes.c_int64 * 2)()
    L = _lib.lib()
    _lib.check(L.sv_plan_program(n, packed.ptr, packed.n, None, 0, None, 0, sizes))
    ints = np.zeros(sizes[0], dtype=np.int64)
    dbls = np.zeros(max(sizes[1], 1), dtype=np.float64)
    _lib.check(L.sv_plan_program(n, packed.ptr, packed.n, ints.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)),
                                 sizes[0], dbls.ctypes.data_as(ctypes.POINTER(ctypes.c_double)), sizes[1], sizes))
    return parse(ints, dbls[: sizes[1]])


def parse(I, D):
    pos = [0]

    def nxt(k=1):
        v = I[pos[0]:pos[0] + k]
        pos[0] += k
        return [int(x) for x in v] if k > 1 else int(v[0])

    C = D[0::2] + 1j * D[1::2]
    assert nxt() == 1
    nl = nxt()
    steps = []
    for _ in range(nxt()):
        if nxt():
            b = nxt()
            tpos = nxt(b) if b > 1 else [nxt()]
            tpos_st = nxt(b) if b > 1 else [nxt()]
            q = nxt(b) if b > 1 else [nxt()]
            steps.append(("pass", dict(b=b, tpos=tpos, tpos_st=tpos_st, q=q, phase_begin=nxt(), n_phases=nxt())))
        else:
            t, fmask, fval, xmask, nb = (nxt() for _ in range(5))
            pp = [nxt() for _ in range(nb)]
            moff, mlen = nxt(), nxt()
            steps.append(("single", dict(type=t, fmask=fmask & 0xFFFFFFFFFFFFFFFF, fval=fval & 0xFFFFFFFFFFFFFFFF,
                                         xmask=xmask & 0xFFFFFFFFFFFFFFFF, nb=nb, pos=pp,
                                         m=C[moff:moff + mlen])))
    phases = []
    for _ in range(nxt()):
        reg = [nxt() for _ in range(KRB)]
        flip = nxt()
        thr = [nxt() for _ in range(KMAXB)]
        phases.append(dict(reg=reg, flip=flip, thr=thr, op_begin=nxt(), op_end=nxt()))
    ops = []
    for _ in range(nxt()):
        pm, pv, xm, fpm, fpv, fk, cs, cm, cv, k, v, xr, nt, mtype = (nxt() for _ in range(14))
        treg = [nxt() for _ in range(6)]
        tphys = [nxt() for _ in range(6)]
        tab, coff = nxt(), nxt()
        ops.append(dict(pm=pm, pv=pv, xm=xm & 0xFFFFFFFFFFFFFFFF, fpm=fpm, fpv=fpv, fk=fk, cs=cs, cm=cm, cv=cv, k=k, v=v, xr=xr, nt=nt, mtype=mtype, treg=treg,
                        tphys=tphys, tab=tab, c=C[coff:coff + 4]))
    coef_off, ncoef = nxt(), nxt()
    coef = C[coef_off:coef_off + ncoef]
    perm = [nxt() for _ in range(nl)]
    return dict(nl=nl, steps=steps, phases=phases, ops=ops, coef=coef, perm=perm)


def _spread(vals, positions):
    out = np.zeros_like(vals, dtype=np.int64)
    for j, p in enumerate(positions):
        out |= ((vals >> j) & 1) << p
    return out


def _insert_zeros(t, positions):
    t = t.astype(np.int64)
    for p in sorted(positions):
        lo = t & ((1 << p) - 1)
        t = ((t ^ lo) << 1) | lo
    return t


def _run_single(state, p, nl):
    idx = np.arange(1 << nl, dtype=np.int64)
    sel = (idx & p["fmask"]) == p["fval"]
    if p["type"] == 0:       # PAIR
        i0 = idx[sel]
        i1 = i0 ^ p["xmask"]
        m = p["m"]
        a0, a1 = state[i0].copy(), state[i1].copy()
        state[i0] = m[0] * a0 + m[1] * a1
        state[i1] = m[2] * a0 + m[3] * a1
    elif p["type"] == 1:     # DIAG
        i = idx[sel]
        t = np.zeros_like(i)
        for j, q in enumerate(p["pos"]):
            t |= ((i >> q) & 1) << j
        state[i] *= p["m"][t]
    else:                    # DENSE
        k = p["nb"]
        base = idx[sel]
        d = 1 << k
        offs = np.array([sum(((r >> j) & 1) << q for j, q in enumerate(p["pos"])) for r in range(d)])
        M = p["m"].reshape(d, d)
        grp = base[:, None] | offs[None, :]
        state[grp] = state[grp] @ M.T


def _run_pass(state, P, prog, nl):
    b = P["b"]
    nthr = b - KRB
    T = 1 << b
    n_tiles = 1 << (nl - b)
    tiles = np.arange(n_tiles, dtype=np.int64)
    base = _insert_zeros(tiles, P["tpos"])                               # (n_tiles,)
    s_all = np.arange(T, dtype=np.int64)
    gidx = base[:, None] | _spread(s_all, P["tpos"])[None, :]            # load addresses
    tile = state[gidx]                                                   # (n_tiles, T)
    tids = np.arange(1 << nthr, dtype=np.int64)
    for ph in prog["phases"][P["phase_begin"]:P["phase_begin"] + P["n_phases"]]:
        thr = ph["thr"][:nthr]
        sthr = _spread(tids, thr)                                        # tile index of r = 0
        phys_base = base[:, None] | _spread(tids, [P["tpos"][t] for t in thr])[None, :]
        regoff = np.array([sum(((r >> k) & 1) << ph["reg"][k] for k in range(KRB)) for r in range(16)])
        a = tile[:, sthr[:, None] | regoff[None, :]]                     # (n_tiles, nthreads, 16)
        fthr = np.zeros(phys_base.shape, dtype=np.int64)
        for op in prog["ops"][ph["op_begin"]:ph["op_end"]]:
            if op["fk"]:   # attached thread-predicated X: toggle the flip before the op
                fthr ^= np.where((phys_base & op["fpm"]) == op["fpv"], op["fk"], 0)
            pred = (phys_base & op["pm"]) == op["pv"]
            _apply(a, op, pred, fthr, phys_base, prog["coef"])
        fl = ph["flip"] ^ fthr                                           # per thread
        for r in range(16):
            dst = sthr[None, :] | _regoff_dyn(r ^ fl, ph["reg"])
            np.put_along_axis(tile, dst.reshape(n_tiles, -1), a[:, :, r].reshape(n_tiles, -1), axis=1)
    # store with the in-tile relabeling: tile index s -> physical bits tpos_st
    sidx = base[:, None] | _spread(s_all, P["tpos_st"])[None, :]
    state[sidx] = tile


def _regoff_dyn(rr, reg):
    out = np.zeros_like(rr)
    for k in range(KRB):
        out |= ((rr >> k) & 1) << reg[k]
    return out


def _apply(a, op, pred, fthr, phys_base, coef):
    cs = op["cs"]
    c = op["c"]

    def pair(r0, r1, m, where):
        x, y = a[..., r0].copy(), a[..., r1].copy()
        m = [np.broadcast_to(mm, where.shape) for mm in m]
        a[..., r0] = np.where(where, m[0] * x + m[1] * y, x)
        a[..., r1] = np.where(where, m[2] * x + m[3] * y, y)

    if CS_PAIR1 <= cs < CS_PAIR1 + 16 or CS_PAIR1D <= cs < CS_PAIR1D + 16:
        k = op["k"]
        if cs >= CS_PAIR1D:
            sw = ((fthr >> k) & 1).astype(bool)
            m = [np.where(sw, c[3], c[0]), np.where(sw, c[2], c[1]), np.where(sw, c[1], c[2]),
                 np.where(sw, c[0], c[3])]
        else:
            m = list(c)
        for r in range(16):
            if not (r >> k) & 1:
                pair(r, r | (1 << k), m, pred)
    elif CS_SHEAR <= cs < CS_SHEAR + 16:
        k, kind = (cs - CS_SHEAR) // 4, (cs - CS_SHEAR) % 4
        t, s = c[0].real, c[0].imag
        if kind == 2:
            sg = np.where(((fthr >> k) & 1).astype(bool), -1.0, 1.0)
            t, s = sg * t, sg * s

        def shear(u, v, t, s):   # u += t v; v += s u; u += t v   (same rounding as the kernel's FMAs)
            u = u + t * v
            v = v + s * u
            return u + t * v, v

        for r in range(16):
            if (r >> k) & 1:
                continue
            x0, x1 = a[..., r].copy(), a[..., r | (1 << k)].copy()
            if kind == 1:
                ure, vim = shear(x0.real, x1.imag, -t, -s)
                uim, vre = shear(x0.imag, x1.real, t, s)
                n0, n1 = ure + 1j * uim, vre + 1j * vim
            else:
                r0, r1 = shear(x0.real, x1.real, t, s)
                i0, i1 = shear(x0.imag, x1.imag, t, s)
                n0, n1 = r0 + 1j * i0, r1 + 1j * i1
            a[..., r] = np.where(pred, n0, x0)
            a[..., r | (1 << k)] = np.where(pred, n1, x1)
    elif CS_TAN <= cs < CS_TAND + 8:
        if cs >= CS_TAND:
            k, kind = (cs - CS_TAND) // 2, 2 * ((cs - CS_TAND) % 2)
            neg = ((fthr >> k) & 1).astype(bool)
        else:
            k, kind = (cs - CS_TAN) // 4, (cs - CS_TAN) % 4
            neg = np.zeros_like(pred, dtype=bool)
        t = c[0].real
        # flipped roles = R(-phi): TAN negates t; COT negates the +-1 terms (R(-phi) = s[[k, 1], [-1, k]])
        tt = np.where(neg, -t, t) if kind == 0 else t
        one = np.where(neg, -1.0, 1.0)
        for r in range(16):
            if (r >> k) & 1:
                continue
            x0, x1 = a[..., r].copy(), a[..., r | (1 << k)].copy()
            if kind == 0:     # x0 - t x1, x1 + t x0
                n0, n1 = x0 - tt * x1, x1 + tt * x0
            elif kind == 1:   # x0 - i t x1, x1 - i t x0
                n0, n1 = x0 - 1j * t * x1, x1 - 1j * t * x0
            elif kind == 2:   # t x0 - x1, t x1 + x0
                n0, n1 = t * x0 - one * x1, t * x1 + one * x0
            else:             # t x0 - i x1, t x1 - i x0
                n0, n1 = t * x0 - 1j * x1, t * x1 - 1j * x0
            a[..., r] = np.where(pred, n0, x0)
            a[..., r | (1 << k)] = np.where(pred, n1, x1)
    elif CS_PARITY <= cs < CS_PARITY + 16:
        M = cs - CS_PARITY
        popc = np.vectorize(lambda x: bin(int(x)).count("1"))
        tp = (popc(phys_base & op["xm"]) + popc(fthr & M) + op["v"]) & 1
        for r in range(16):
            hit = pred & (((bin(r & M).count("1") & 1) ^ tp) == 1)
            a[..., r] = np.where(hit, c[0] * a[..., r], a[..., r])
    elif CS_PHASE1 <= cs < CS_PHASE1 + 8 or CS_PHASE1D <= cs < CS_PHASE1D + 8:
        k = op["k"]
        v = op["v"] ^ (((fthr >> k) & 1) if cs >= CS_PHASE1D else 0)
        for r in range(16):
            hit = pred & (((r >> k) & 1) == v)
            a[..., r] = np.where(hit, c[0] * a[..., r], a[..., r])
    elif cs == CS_RDIAG:
        for r in range(16):
            if (op["xm"] >> r) & 1:
                a[..., r] = np.where(pred, coef[op["tab"] + r] * a[..., r], a[..., r])
    elif cs == CS_SCALAR:
        for r in range(16):
            a[..., r] = np.where(pred, c[0] * a[..., r], a[..., r])
    elif CS_XFLIP <= cs < CS_XFLIP + 4:
        fthr ^= np.where(pred, 1 << op["k"], 0)
    elif CS_PAIRGR <= cs < CS_PAIRG + 15:
        xr = op["xr"]
        cv = op["cv"] ^ (fthr & op["cm"])
        for r in range(16):
            pair(r, r ^ xr, list(c), pred & ((r & op["cm"]) == cv))
    elif cs == CS_DIAGG:
        tconst = np.zeros(pred.shape, dtype=np.int64)
        w = [0, 0, 0, 0]
        for j in range(op["nt"]):
            rg = op["treg"][j]
            if rg == 0xFF:
                tconst |= ((phys_base >> op["tphys"][j]) & 1) << j
            else:
                tconst ^= ((fthr >> rg) & 1) << j
                w[rg] |= 1 << j
        cv = op["cv"] ^ (fthr & op["cm"])
        for r in range(16):
            t = tconst ^ sum(w[k] for k in range(KRB) if (r >> k) & 1)
            hit = pred & ((r & op["cm"]) == cv)
            a[..., r] = np.where(hit, coef[op["tab"] + t] * a[..., r], a[..., r])
    elif CS_DENSE2 <= cs < CS_DENSE2 + 6:
        k0, k1 = op["xr"] & 15, op["xr"] >> 4
        f = ((fthr >> k0) & 1) | (((fthr >> k1) & 1) << 1)
        cv = op["cv"] ^ (fthr & op["cm"])
        M = coef[op["tab"]:op["tab"] + 16]
        B0, B1 = 1 << k0, 1 << k1
        for r in range(16):
            if r & (B0 | B1):
                continue
            hit = pred & ((r & op["cm"]) == cv)
            idx = [r, r | B0, r | B1, r | B0 | B1]
            v = [a[..., i].copy() for i in idx]
            for qq in range(4):
                acc = sum(M[((qq ^ f) * 4 + (cc ^ f))] * v[cc] for cc in range(4))
                a[..., idx[qq]] = np.where(hit, acc, a[..., idx[qq]])
    else:
        raise AssertionError(f"unknown case {cs}")


def run_program(prog, state):
    """Execute the planned program on ``state`` (physical layout) and return the state in the
    canonical (identity) layout."""
    nl = prog["nl"]
    st = np.array(state, dtype=np.complex128)
    for kind, item in prog["steps"]:
        if kind == "pass":
            _run_pass(st, item, prog, nl)
        else:
            _run_single(st, item, nl)
    # qubit at physical p moved to perm[p]: canonical index bit p <- physical bit perm[p]
    idx = np.arange(1 << nl, dtype=np.int64)
    phys = np.zeros_like(idx)
    for p in range(nl):
        phys |= ((idx >> p) & 1) << prog["perm"][p]
    return st[phys]
