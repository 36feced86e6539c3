"""Host mirror of the device page layout (csrc/sk_layout.cuh, csrc/sk_common.cuh).

Used only to *read* device pages back into the reference's PhysicalPage
view (codes, scale/zero, stats) -- the device kernels write and consume the
layout themselves.  Index maps are cached per geometry.
"""

from __future__ import annotations

import functools

import numpy as np


def code_row_bytes(head_dim: int, bits: int) -> int:
    return head_dim * 2 if bits == 0 else (head_dim // 2 if bits <= 4 else head_dim)


def slot_bytes(head_dim: int, page: int, bits: int) -> int:
    b = 2 * page * code_row_bytes(head_dim, bits) + (8 * head_dim if bits else 0)
    return (b + 127) // 128 * 128


def _kparts(d):
    s, h, j, e = d // 16, (d % 16) // 8, (d % 8) // 2, d % 2
    return s, h, j, e, 2 * s + h


def _vparts(t, c):
    cn, c8 = c // 8, c % 8
    ks, h, j, e = t // 16, (t % 16) // 8, (t % 8) // 2, t % 2
    return cn, 4 * c8 + j, 2 * ks + h, e


@functools.lru_cache(maxsize=None)
def maps(head_dim: int, page: int, bits: int):
    """Return (k_index, v_index, k_shift, v_shift) arrays of shape [P, D].

    bits <= 4: byte offsets + nibble shift; 5..8: byte offsets; 0: element
    offsets (16-bit values) -- each relative to the K or V region start."""
    D, P = head_dim, page
    t = np.arange(P)[:, None].repeat(D, 1)
    d = np.arange(D)[None, :].repeat(P, 0)
    s, h, j, e, ri = _kparts(d)
    cn, lane, vri, ve = _vparts(t, d)
    if bits == 0:
        k_idx = t * D + j * (D // 4) + ri * 2 + e
        v_idx = (cn * 32 + lane) * (P // 4) + vri * 2 + ve
        return k_idx, v_idx, None, None
    if bits <= 4:
        w, slot = ri // 4, ri % 4
        bit = 4 * slot + 16 * e
        k_idx = t * (D // 2) + j * (D // 8) + w * 4 + bit // 8
        k_sh = bit % 8
        vw, vslot = vri // 4, vri % 4
        vbit = 4 * vslot + 16 * ve
        v_idx = (cn * 32 + lane) * (P // 8) + vw * 4 + vbit // 8
        v_sh = vbit % 8
        return k_idx, v_idx, k_sh, v_sh
    k_idx = t * D + j * (D // 4) + ri * 2 + e
    v_idx = (cn * 32 + lane) * (P // 4) + vri * 2 + ve
    return k_idx, v_idx, None, None


@functools.lru_cache(maxsize=None)
def bound_maps(head_dim: int):
    D = head_dim
    d = np.arange(D)
    s, h, j, e, ri = _kparts(d)
    kpos = j * (D // 4) + ri * 2 + e
    cn, jj, ee = d // 8, (d % 8) // 2, d % 2
    vpos = jj * (D // 4) + cn * 2 + ee
    return kpos, vpos


def decode_slot(raw: np.ndarray, head_dim: int, page: int, bits: int, np_dtype):
    """Unpack one slot's bytes -> (k_codes, v_codes, k_lo, k_hi, v_lo, v_hi).

    Codes are uint8 [P, D] (bits > 0) or np_dtype values [P, D] (bits == 0);
    bounds are np_dtype [D] in natural channel order (None for bits == 0)."""
    D, P = head_dim, page
    rb = code_row_bytes(D, bits)
    kreg = raw[:P * rb]
    vreg = raw[P * rb:2 * P * rb]
    k_idx, v_idx, k_sh, v_sh = maps(D, P, bits)
    if bits == 0:
        kv = kreg.view(np_dtype)
        vv = vreg.view(np_dtype)
        return kv[k_idx], vv[v_idx], None, None, None, None
    if bits <= 4:
        kc = (kreg[k_idx] >> k_sh) & 0xF
        vc = (vreg[v_idx] >> v_sh) & 0xF
    else:
        kc = kreg[k_idx]
        vc = vreg[v_idx]
    bnd = raw[2 * P * rb:2 * P * rb + 8 * D].view(np_dtype).reshape(4, D)
    kpos, vpos = bound_maps(D)
    return (kc.astype(np.uint8), vc.astype(np.uint8), bnd[0][kpos], bnd[1][kpos], bnd[2][vpos], bnd[3][vpos])


def encode_slot(kc, vc, klo, khi, vlo, vhi, head_dim: int, page: int, bits: int, np_dtype, slot_bytes: int):
    """Inverse of decode_slot: pack one page (codes [t, D] for t <= P tokens,
    bounds [D] in natural channel order) into the device slot layout."""
    D, P = head_dim, page
    rb = code_row_bytes(D, bits)
    raw = np.zeros(slot_bytes, np.uint8)
    t = kc.shape[0]
    k_idx, v_idx, k_sh, v_sh = maps(D, P, bits)
    if bits == 0:
        kreg = np.zeros(P * D, np_dtype)
        vreg = np.zeros(P * D, np_dtype)
        kreg[k_idx[:t]] = kc
        vreg[v_idx[:t]] = vc
        raw[:P * rb] = kreg.view(np.uint8)
        raw[P * rb:2 * P * rb] = vreg.view(np.uint8)
        return raw
    kreg = np.zeros(P * rb, np.uint8)
    vreg = np.zeros(P * rb, np.uint8)
    if bits <= 4:
        np.bitwise_or.at(kreg, k_idx[:t].ravel(), (kc.astype(np.uint8) << k_sh[:t]).ravel().astype(np.uint8))
        np.bitwise_or.at(vreg, v_idx[:t].ravel(), (vc.astype(np.uint8) << v_sh[:t]).ravel().astype(np.uint8))
    else:
        kreg[k_idx[:t]] = kc
        vreg[v_idx[:t]] = vc
    raw[:P * rb] = kreg
    raw[P * rb:2 * P * rb] = vreg
    kpos, vpos = bound_maps(D)
    bnd = np.zeros((4, D), np_dtype)
    bnd[0][kpos], bnd[1][kpos], bnd[2][vpos], bnd[3][vpos] = klo, khi, vlo, vhi
    raw[2 * P * rb:2 * P * rb + 8 * D] = bnd.view(np.uint8).ravel()
    return raw
