"""Generate the golden fixtures in tests/golden/ from the REFERENCE itself.

Runs the unmodified reference headers compiled by oracle/Makefile
(oracle/_ref/libmdreg_ref.so, built from /root/reference/proj) on small seeded
inputs and stores inputs + outputs as .npz.  The fixtures pin both the C
restatement (tests/test_oracle.py, CPU) and the CUDA path (tests/test_gpu_*.py)
without needing /root/reference at test time.

    python tests/golden/make_golden.py      # needs /root/reference
"""
from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
from _util import f32, random_field, random_feature_map, random_qk  # noqa: E402

import pyoracle  # noqa: E402


def attention_case(ref, dims, S, hd, nb, seed):
    h, w, l = dims
    n = h * w * l
    Q = random_qk(dims, S * hd, seed)
    K = random_qk(dims, S * hd, seed + 1)
    B = f32(pyoracle.Rng(seed + 2).normal(S * nb ** 3).reshape(S, nb ** 3))
    W, err = ref.na_fwd(Q, K, B, dims, S, hd, nb)
    assert err is None, err
    SF = ref.subfields_fwd(W, dims, S, nb)
    gSF = f32(pyoracle.Rng(seed + 3).normal(3 * S * n).reshape(SF.shape))
    gW = ref.subfields_bwd(gSF, dims, S, nb)
    gQ, gK, gB = ref.na_bwd(Q, K, W, gW, dims, S, hd, nb)
    return dict(dims=np.array(dims), S=S, hd=hd, nb=nb, Q=Q, K=K, B=B, W=W, SF=SF, gSF=gSF,
                gW=gW, gQ=gQ, gK=gK, gB=gB)


def warp_case(ref, dims, C, mag, seed):
    vol = random_feature_map(C, dims, seed)
    fld = random_field(dims, seed + 1, mag)
    out = ref.warp_fwd(vol, fld)
    gout = random_feature_map(C, dims, seed + 2)
    gin, gfield = ref.warp_bwd(vol, fld, gout)
    return dict(dims=np.array(dims), vol=vol, field=fld, out=out, gout=gout, gin=gin,
                gfield=gfield)


def main():
    if not pyoracle.ref_available():
        pyoracle.build()
    ref = pyoracle.ref()
    out = {}
    out["attn_7x6x5_s2_d4"] = attention_case(ref, (7, 6, 5), 2, 4, 3, 100)
    out["attn_6x5x4_s1_d6"] = attention_case(ref, (6, 5, 4), 1, 6, 3, 110)
    out["attn_5x4x3_s1_d3_nb5"] = attention_case(ref, (5, 4, 3), 1, 3, 5, 120)
    out["attn_1x1x1_s1_d3"] = attention_case(ref, (1, 1, 1), 1, 3, 3, 130)
    out["attn_2x1x3_s3_d2"] = attention_case(ref, (2, 1, 3), 3, 2, 3, 140)
    out["warp_7x6x5_c3_m1p5"] = warp_case(ref, (7, 6, 5), 3, 1.5, 200)
    out["warp_6x5x4_c2_m6"] = warp_case(ref, (6, 5, 4), 2, 6.0, 210)   # heavy clamping
    out["warp_5x1x4_c1_m1"] = warp_case(ref, (5, 1, 4), 1, 1.0, 220)   # collapsed axis

    # upsample: doubling-range targets incl. 2d-1 and 2d+1
    for name, d, td in (("up_4x3x3_to_8x6x5", (4, 3, 3), (8, 6, 5)),
                        ("up_4x4x4_to_7x8x9", (4, 4, 4), (7, 8, 9)),
                        ("up_1x2x2_to_2x3x4", (1, 2, 2), (2, 3, 4))):
        x = random_feature_map(3, d, 300 + len(out))
        y = ref.upsample2_fwd(x, td, 2.0)
        g = random_feature_map(3, td, 400 + len(out))
        gin = ref.upsample2_bwd(g, d, 2.0)
        out[name] = dict(dims=np.array(d), tdims=np.array(td), x=x, y=y, gout=g, gin=gin)

    # RegHead-shaped conv3 (ic = 3S = 6, oc = 3) with a zero tap
    d = (6, 5, 4)
    x = random_feature_map(6, d, 500)
    k = f32(pyoracle.Rng(501).normal(3 * 6 * 27, 0.0, 0.3).reshape(3, 6, 3, 3, 3))
    k[0, 0, 1, 1, 1] = 0.0
    b = f32(pyoracle.Rng(502).normal(3))
    y = ref.conv3_fwd(x, k, b)
    g = random_feature_map(3, d, 503)
    gin, gk, gb = ref.conv3_bwd(x, k, g)
    out["conv3_6x5x4_ic6_oc3"] = dict(dims=np.array(d), x=x, k=k, b=b, y=y, gout=g, gin=gin,
                                      gk=gk, gb=gb)

    # compose and scaling-squaring
    d = (7, 6, 5)
    prev = random_field(d, 600, 1.2)
    res = random_field(d, 601, 0.8)
    c = ref.compose_fwd(prev, res)
    g = random_feature_map(3, d, 602)
    gp, gr = ref.compose_bwd(prev, res, g)
    out["compose_7x6x5"] = dict(dims=np.array(d), prev=prev, res=res, out=c, gout=g, gprev=gp,
                                gres=gr)
    v = ref.make_smooth_velocity((8, 7, 6), 11, 2.0, 2.0)
    out["ss_8x7x6_t7"] = dict(dims=np.array((8, 7, 6)), vel=v, out=ref.scaling_squaring(v, 7))

    for name, arrs in out.items():
        np.savez_compressed(os.path.join(HERE, name + ".npz"), **arrs)
    total = sum(os.path.getsize(os.path.join(HERE, n + ".npz")) for n in out)
    print(f"wrote {len(out)} fixtures, {total / 1e3:.1f} kB")


if __name__ == "__main__":
    main()
