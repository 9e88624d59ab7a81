"""Generate golden vectors by running the REFERENCE package itself.

Run in the build container (where /root/reference exists):

    python tests/golden/make_golden.py

It imports `bandred` read-only from /root/reference/pkg/src (bytecode writes
disabled), runs its public functions on small seeded inputs, and stores
inputs + outputs in tests/golden/*.npz. These fixtures pin both the NumPy
oracle (tests/test_oracle_golden.py, CPU) and the CUDA path
(tests/test_gpu_parity.py, GPU). /root/reference is never read at test time.
"""
import os
import sys
import warnings

sys.dont_write_bytecode = True
REF = os.environ.get("BANDRED_REF_SRC", "/root/reference/pkg/src")
sys.path.insert(0, REF)

import numpy as np  # noqa: E402
import bandred  # noqa: E402
from bandred import kernels as K  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))


def rand(m, n, seed):
    return np.asfortranarray(np.random.default_rng(seed).standard_normal((m, n)))


def sym(n, seed):
    g = np.random.default_rng(seed).standard_normal((n, n))
    return np.asfortranarray((g + g.T) / 2.0)


def poison_upper(A):
    A = A.copy(order="F")
    A[np.triu_indices(A.shape[0], 1)] = 1e9
    return A


def kernels_golden():
    d = {}
    # house_gen known answers (pkg/tests/test_kernels.py:147-181) + random
    hcases = {
        "h345": np.array([3.0, 4.0]),
        "hzero": np.zeros(4),
        "hzerotail": np.array([2.0, 0.0, 0.0]),
        "hneg1": np.array([-3.0]),
        "hx0zero": np.array([0.0, 1.0, -2.0]),
        "hrand": np.random.default_rng(21).standard_normal(37),
    }
    for name, x in hcases.items():
        v, tau, beta = bandred.house_gen(x)
        d[f"{name}_x"] = x
        d[f"{name}_v"] = v
        d[f"{name}_tb"] = np.array([tau, beta])

    # qr / lq panels: random, square, zero column, already triangular, tall
    qr_cases = {
        "qr_40x6": rand(40, 6, 100),
        "qr_sq8": rand(8, 8, 101),
        "qr_257x32": rand(257, 32, 102),
        "qr_300x40": rand(300, 40, 103),  # crosses inner_b=16 blocks, 40 > 32
        "qr_tri": np.asfortranarray(np.vstack([np.triu(rand(5, 5, 104)), np.zeros((7, 5))])),
    }
    zc = rand(64, 8, 105)
    zc[:, 3] = 0.0
    qr_cases["qr_zerocol"] = zc
    for name, P in qr_cases.items():
        Pw = P.copy(order="F")
        f = K.qr_panel(Pw)
        d[f"{name}_in"] = P
        d[f"{name}_Y"], d[f"{name}_T"], d[f"{name}_W"] = f.y, f.t, f.w
        d[f"{name}_R"], d[f"{name}_tau"], d[f"{name}_out"] = f.r_or_l, f.tau, Pw
    lq_cases = {
        "lq_6x40": rand(6, 40, 110),
        "lq_32x257": rand(32, 257, 111),
        "lq_sq8": rand(8, 8, 112),
    }
    for name, P in lq_cases.items():
        Pw = P.copy(order="F")
        f = K.lq_panel(Pw)
        d[f"{name}_in"] = P
        d[f"{name}_Y"], d[f"{name}_T"], d[f"{name}_W"] = f.y, f.t, f.w
        d[f"{name}_L"], d[f"{name}_tau"], d[f"{name}_out"] = f.r_or_l, f.tau, Pw

    # WY application
    f = K.qr_panel(rand(100, 8, 120))
    A0 = rand(100, 37, 121)
    A = A0.copy(order="F")
    K.apply_wy_left(A, f)
    d.update(awl_Y=f.y, awl_W=f.w, awl_in=A0, awl_out=A)
    f = K.lq_panel(rand(8, 90, 122))
    A0 = rand(45, 90, 123)
    A = A0.copy(order="F")
    K.apply_wy_right(A, f)
    d.update(awr_Y=f.y, awr_W=f.w, awr_in=A0, awr_out=A)

    # symmetric kernels with a poisoned upper triangle (test_kernels.py:356-377)
    S = poison_upper(sym(150, 130))
    Wm = rand(150, 12, 131)
    X1 = np.zeros((150, 12), order="F")
    K.symm_lower(S, Wm, X1)
    d.update(symm_A=S, symm_W=Wm, symm_X1=X1)
    S0 = poison_upper(sym(140, 132))
    X3 = rand(140, 10, 133)
    Ym = rand(140, 10, 134)
    Sw = S0.copy(order="F")
    K.syr2k_lower(Sw, X3, Ym, 0, 140)
    Sp = S0.copy(order="F")
    K.syr2k_lower(Sp, X3, Ym, 37, 101)
    d.update(syr_A=S0, syr_X3=X3, syr_Y=Ym, syr_out=Sw, syr_part_out=Sp)
    f = K.qr_panel(rand(120, 9, 135))
    S0 = poison_upper(sym(120, 136))
    Sw = S0.copy(order="F")
    K.sym_two_sided_update(Sw, f)
    d.update(tsu_A=S0, tsu_Y=f.y, tsu_W=f.w, tsu_out=Sw)
    np.savez_compressed(os.path.join(OUT, "kernels.npz"), **d)
    print("kernels.npz", len(d), "arrays")


SEVP_CASES = [
    # (name, n, w, b, seed, variant)
    ("s64_8_8", 64, 8, 8, 200, "reference"),
    ("s100_12_5", 100, 12, 5, 201, "reference"),  # b < w, fringe panel
    ("s130_16_16", 130, 16, 16, 202, "v2"),  # (n-w) mod b = 2
    ("s97_16_16", 97, 16, 16, 203, "reference"),  # (n-w) mod b = 1
    ("s256_32_32", 256, 32, 32, 204, "v2"),  # c1 shape at n=256
    ("s200_40_10", 200, 40, 10, 205, "v1"),
    ("s300_64_64", 300, 64, 64, 206, "reference"),
]

TRI_CASES = [
    # (name, m, n, w, b, seed)
    ("t64_8_8", 64, 64, 8, 8, 300),
    ("t100_80_12_5", 100, 80, 12, 5, 301),
    ("t70_90_6_6", 70, 90, 6, 6, 302),  # wide: reduces the transpose
    ("t256_32_32", 256, 256, 32, 32, 303),
    ("t97_16_16", 97, 97, 16, 16, 304),
    ("t300_64_64", 300, 300, 64, 64, 305),
]


def reductions_golden():
    d = {}
    V = {"reference": bandred.SevpVariant.REFERENCE, "v1": bandred.SevpVariant.V1,
         "v2": bandred.SevpVariant.V2}
    for name, n, w, b, seed, var in SEVP_CASES:
        A = poison_upper(sym(n, seed))
        cfg = bandred.SevpConfig(n=n, w=w, b=b, variant=V[var])
        with warnings.catch_warnings():
            warnings.simplefilter("ignore")
            res = bandred.reduce_sym_band(A, cfg)
        d[f"{name}_A"] = A
        d[f"{name}_band"] = res.band
        d[f"{name}_meta"] = np.array([n, w, b, res.iterations, res.flops["total"]], dtype=np.int64)
    # accumulate_q case
    A = sym(48, 207)
    res = bandred.reduce_sym_band(A, bandred.SevpConfig(n=48, w=6, b=3, accumulate_q=True))
    d.update(sq_A=A, sq_band=res.band, sq_Q=res.q)
    for name, m, n, w, b, seed in TRI_CASES:
        A = rand(m, n, seed)
        res = bandred.reduce_tri_band(A, w, b)
        d[f"{name}_A"] = A
        d[f"{name}_band"] = res.band
        d[f"{name}_meta"] = np.array([m, n, w, b, res.iterations, res.flops["total"],
                                      res.lower_bw, res.upper_bw], dtype=np.int64)
    np.savez_compressed(os.path.join(OUT, "reductions.npz"), **d)
    print("reductions.npz", len(d), "arrays")


BAND_CASES = [
    # (name, m, n, w, b, seed, variant)
    ("b64_8_8_ref", 64, 64, 8, 8, 400, "reference"),
    ("b64_8_8_sim", 64, 64, 8, 8, 400, "simultaneous"),
    ("b64_8_8_v2", 64, 64, 8, 8, 400, "v2"),
    ("b80_12_4_v1", 80, 80, 12, 4, 401, "v1"),
    ("b80_12_4_ref", 80, 80, 12, 4, 401, "reference"),
    ("b96_70_8_6_ref", 96, 70, 8, 6, 402, "reference"),  # rectangular m > n
    ("b50_90_6_6_sim", 50, 90, 6, 6, 403, "simultaneous"),  # wide: transpose
    ("b256_32_32_v2", 256, 256, 32, 32, 404, "v2"),
    ("b130_16_16_ref", 130, 130, 16, 16, 405, "reference"),
]


def band_golden():
    d = {}
    V = {"reference": bandred.SvdVariant.REFERENCE, "simultaneous": bandred.SvdVariant.SIMULTANEOUS,
         "v1": bandred.SvdVariant.V1, "v2": bandred.SvdVariant.V2}
    for name, m, n, w, b, seed, var in BAND_CASES:
        A = rand(m, n, seed)
        cfg = bandred.SvdConfig(m=m, n=n, w=w, b=b, form=bandred.SvdForm.BAND, variant=V[var])
        with warnings.catch_warnings():
            warnings.simplefilter("ignore")
            res = bandred.reduce_band_svd(A, cfg)
        d[f"{name}_A"] = A
        d[f"{name}_band"] = res.band
        d[f"{name}_meta"] = np.array([m, n, w, b, res.iterations, res.flops["total"], res.lower_bw,
                                      res.upper_bw], dtype=np.int64)
    np.savez_compressed(os.path.join(OUT, "band.npz"), **d)
    print("band.npz", len(d), "arrays")


def cli_golden():
    """SplitMix64 inputs and the text matrix format of the reference CLI."""
    from bandred import cli

    d = {"gen_general_7_5_9": cli.gen_general(7, 5, 9), "gen_sym_6_3": cli.gen_sym(6, 3),
         "gen_general_33_17_123456789": cli.gen_general(33, 17, 123456789)}
    np.savez_compressed(os.path.join(OUT, "cli.npz"), **d)
    A = cli.gen_general(4, 3, 2) * 1e6 - 5e5
    A[1, 1] = -0.0
    A[2, 0] = 1e-300
    d2 = os.path.join(OUT, "matrix_4x3.txt")
    cli.save_matrix(d2, A)
    print("cli.npz", len(d), "arrays; matrix_4x3.txt")


if __name__ == "__main__":
    kernels_golden()
    reductions_golden()
    band_golden()
    cli_golden()
