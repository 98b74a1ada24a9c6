"""NumPy emulator of the tile-pass kernel (qsv_tile_block.cu) -- TEST
INFRASTRUCTURE ONLY.

Executes the program the native planner compiles (exported through
qsv_debug_plan_json) with the kernel's exact data movement: tiles gathered
through offhi/comp, SMEM slots through the swizzle and the per-block
GF(2)-affine map, register blocks vectorised over cosets, and the final store
through the pass's map.  Lets tests check the planner and its encoding on CPU
against the oracle.
"""

from __future__ import annotations

import numpy as np

OP_U1, OP_U2, OP_CX, OP_SWAP, OP_X, OP_DIAG1, OP_ROTG, OP_ROTD, OP_GMAT, OP_U1C = 1, 2, 3, 4, 5, 6, 7, 8, 9, 10


def swz(l):
    """Tile swizzle (qsv_internal.h tile_swz): bits 0..2 = (l ^ F) & 7, bits
    3..5 = F, F = fold of the higher 3-bit chunks."""
    f = ((l >> 3) ^ (l >> 6) ^ (l >> 9)) & 7
    return (l & ~63) | (f << 3) | ((l ^ f) & 7)


def popc(x):
    return np.bitwise_count(np.asarray(x, dtype=np.uint64)).astype(np.int64)


def _c(params, p, k):
    return complex(params[p + 2 * k], params[p + 2 * k + 1])


def _rot_coeffs(rot):
    s_hi, s_loc, q, c, s = rot
    kk = -s if (q & 2) else s
    imag = bool(q & 1)
    return s_hi, s_loc, q, c, kk, imag


def _mix(c, a0, k, imag, a1):
    return c * a0 + (1j * k if imag else k) * a1


def run_block(a, ops, rots, params, tid, base, blk_ops, RB):
    """a: (ncos, 2^RB) complex; tid: (ncos,) thread indices; base: tile base index."""
    R = 1 << RB
    for op in blk_ops:
        typ, oa, ob, oh, r0, r1, p, f = op
        if typ == OP_U1:
            J = 1 << oa
            m00, m01, m10, m11 = (_c(params, p, k) for k in range(4))
            for r in range(R):
                if r & J:
                    continue
                x, y = a[:, r].copy(), a[:, r | J].copy()
                a[:, r] = m00 * x + m01 * y
                a[:, r | J] = m10 * x + m11 * y
        elif typ == OP_U1C:  # 2x2 on bit oa, matrix selected by bit ob
            J = 1 << oa
            for r in range(R):
                if r & J:
                    continue
                q = p + 8 * ((r >> ob) & 1)
                m00, m01, m10, m11 = (_c(params, q, k) for k in range(4))
                x, y = a[:, r].copy(), a[:, r | J].copy()
                a[:, r] = m00 * x + m01 * y
                a[:, r | J] = m10 * x + m11 * y
        elif typ == OP_U2:
            JA, JB = 1 << oa, 1 << ob
            M = np.array([[_c(params, p + 8 * k, i) for i in range(4)] for k in range(4)])
            for r in range(R):
                if r & (JA | JB):
                    continue
                idx = [r, r | JB, r | JA, r | JA | JB]
                x = a[:, idx].copy()
                a[:, idx] = x @ M.T
        elif typ == OP_DIAG1:
            d0, d1 = _c(params, p, 0), _c(params, p, 1)
            if oa >= 0:
                for r in range(R):
                    a[:, r] *= d1 if (r >> oa) & 1 else d0
            else:
                bit = (tid >> ob) & 1
                a *= np.where(bit, d1, d0)[:, None]
        elif typ in (OP_CX, OP_SWAP, OP_X):
            # in-register permutation on block-local bits
            perm = []
            for r in range(R):
                if typ == OP_CX:
                    q = r ^ (1 << ob) if (r >> oa) & 1 else r
                elif typ == OP_SWAP:
                    ba, bb = (r >> oa) & 1, (r >> ob) & 1
                    q = r ^ ((ba ^ bb) * ((1 << oa) | (1 << ob)))
                else:
                    q = r ^ (1 << oa)
                perm.append(q)
            a[:, :] = a[:, perm]
        elif typ == OP_GMAT:
            F = f
            H = F.bit_length() - 1
            w = bin(F).count("1")
            ncfg = 1 << (w - 1)
            s_hi, s_loc, q, c, kk, imag = _rot_coeffs(rots[r0])
            zB = (q >> 8) & (R - 1)
            par0 = (popc(base & s_hi) + popc(tid & (q >> 12))) & 1
            fpos = [j for j in range(RB) if (F >> j) & 1]
            for r in range(R):
                if r & (1 << H):
                    continue
                r1 = r ^ F
                cfg, k = 0, 0
                for j in fpos:
                    if j == H:
                        continue
                    cfg |= ((r1 >> j) & 1) << k
                    k += 1
                cp = par0 ^ (bin(r1 & zB).count("1") & 1)
                idx = p + 8 * (cp * ncfg + cfg)
                m = [np.array([params[i + 2 * e] + 1j * params[i + 2 * e + 1] for i in idx]) for e in range(4)]
                x, y = a[:, r].copy(), a[:, r1].copy()
                a[:, r] = m[0] * x + m[1] * y
                a[:, r1] = m[2] * x + m[3] * y
        elif typ in (OP_ROTG, OP_ROTD):
            for k in range(r0, r1):
                s_hi, s_loc, q, c, kk, imag = _rot_coeffs(rots[k])
                sB = (q >> 8) & (R - 1)
                s_thr = (q >> 12)
                par = (popc(base & s_hi) + popc(tid & s_thr)) & 1
                if typ == OP_ROTD:
                    s = rots[k][4]
                    for r in range(R):
                        sg = par ^ (bin(r & sB).count("1") & 1)
                        ks = np.where(sg, s, -s)
                        a[:, r] = a[:, r] * (c + 1j * ks)
                else:
                    F = f
                    H = F.bit_length() - 1
                    yodd = (q >> 2) & 1
                    for r in range(R):
                        if r & (1 << H):
                            continue
                        r1i = r ^ F
                        s1 = par ^ (bin(r1i & sB).count("1") & 1)
                        s0 = s1 ^ yodd
                        k1 = np.where(s1, -kk, kk)
                        k0 = np.where(s0, -kk, kk)
                        x, y = a[:, r].copy(), a[:, r1i].copy()
                        a[:, r] = _mix(c, x, k1, imag, y)
                        a[:, r1i] = _mix(c, y, k0, imag, x)


def map_slot(l, m, tswz, cols):
    o = tswz
    for b in range(m):
        if (l >> b) & 1:
            o ^= cols[b]
    return o


def run_program(prog: dict, psi: np.ndarray) -> np.ndarray:
    psi = psi.copy()
    ops, rots, params = prog["ops"], prog["rots"], prog["params"]
    n = prog["n"]
    RB = prog.get("block_bits", 4)
    R, TB = 1 << RB, 12 - RB
    for ps in prog["passes"]:
        if ps["global"]:
            flip = ps["flip"]
            h = flip.bit_length() - 1
            j = np.arange(1 << n, dtype=np.int64)
            j0 = j[(j >> h) & 1 == 0]
            j1 = j0 ^ flip
            for op in ops[ps["op_begin"]:ps["op_end"]]:
                for k in range(op[4], op[5]):
                    s_hi, _, q, c, kk, imag = _rot_coeffs(rots[k])
                    s1 = popc(j1 & s_hi) & 1
                    s0 = s1 ^ ((q >> 2) & 1)
                    a0, a1 = psi[j0].copy(), psi[j1].copy()
                    psi[j0] = _mix(c, a0, np.where(s1, -kk, kk), imag, a1)
                    psi[j1] = _mix(c, a1, np.where(s0, -kk, kk), imag, a0)
            continue
        m, pos, comp = ps["m"], ps["pos"], ps["comp"]
        tsize = 1 << m
        loc = np.zeros(tsize, dtype=np.int64)
        for b in range(m):
            loc |= ((np.arange(tsize) >> b) & 1) << pos[b]
        ncos = tsize >> RB
        tid = np.arange(ncos, dtype=np.int64)
        for tile in range(1 << len(comp)):
            base = 0
            for i, q in enumerate(comp):
                if (tile >> i) & 1:
                    base |= 1 << q
            sm = np.zeros(tsize, dtype=np.complex128)
            sm[swz(np.arange(tsize))] = psi[base + loc]
            for blk in ps["blocks"]:
                bops = ops[blk["op0"]:blk["op1"]]
                cols = blk["cols"]
                if blk["kind"] == 0:
                    sb = np.full(ncos, blk["tswz"], dtype=np.int64)
                    for i in range(m - RB):
                        sb ^= np.where((tid >> i) & 1, cols[i], 0)
                    e = cols[TB:TB + RB]
                    off = np.zeros(R, dtype=np.int64)
                    for r in range(R):
                        for j in range(RB):
                            if (r >> j) & 1:
                                off[r] ^= e[j]
                    slots = sb[:, None] ^ off[None, :]
                    a = sm[slots]
                    run_block(a, ops, rots, params, tid, base, bops, RB)
                    sm[slots] = a
                else:
                    typ, oa, ob, oh, r0, r1, p, f = bops[0]
                    for i in range(1 << (m - 1)):
                        l0 = ((i >> oh) << (oh + 1)) | (i & ((1 << oh) - 1))
                        l1 = l0 ^ f
                        p0 = map_slot(l0, m, blk["tswz"], cols)
                        p1 = map_slot(l1, m, blk["tswz"], cols)
                        a0, a1 = sm[p0], sm[p1]
                        for k in range(r0, r1):
                            s_hi, s_loc, q, c, kk, imag = _rot_coeffs(rots[k])
                            s1 = (bin(base & s_hi).count("1") + bin(l1 & s_loc).count("1")) & 1
                            s0 = s1 ^ ((q >> 2) & 1)
                            x, y = a0, a1
                            a0 = _mix(c, x, -kk if s1 else kk, imag, y)
                            a1 = _mix(c, y, -kk if s0 else kk, imag, x)
                        sm[p0], sm[p1] = a0, a1
            # store through the final map
            l = np.arange(tsize)
            st = np.full(tsize, ps["store_t"], dtype=np.int64)
            for b in range(m):
                st ^= np.where((l >> b) & 1, ps["store_cols"][b], 0)
            psi[base + loc] = sm[st]
    return psi
