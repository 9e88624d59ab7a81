"""Golden counted flops for inputs with tau == 0 panel columns, by running
the REFERENCE package itself (build container only; /root/reference is
never read at test time):

    python tests/golden/make_golden_tau0.py

Writes tests/golden/tau0_flops.npz: the inputs and the reference's
`result.flops` totals for SEVP (every variant), the triangular band and the
band form on matrices with exactly-zero panel columns.
"""
import os
import sys

sys.dont_write_bytecode = True
REF = os.environ.get("BANDRED_REF_SRC", "/root/reference/pkg/src")
sys.path.insert(0, REF)

import numpy as np  # noqa: E402
import bandred  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))


def cases():
    # diagonal: every panel column of the SEVP / band form is zero below its
    # diagonal block (tau = 0 throughout)
    yield "diag40", np.asfortranarray(np.diag(np.arange(1.0, 41.0)))
    # a random symmetric matrix with zero rows/columns 5 and 17: zero panel
    # columns in the first iterations only
    g = np.random.default_rng(3).standard_normal((48, 48))
    S = (g + g.T) / 2
    S[[5, 17], :] = 0.0
    S[:, [5, 17]] = 0.0
    yield "zcols48", np.asfortranarray(S)


def main():
    out = {}
    for name, A in cases():
        n = A.shape[0]
        out[f"{name}_A"] = A
        for w, b in ((4, 4), (8, 4), (6, 2)):
            for var in ("REFERENCE", "V1", "V2"):
                if var == "V1" and 2 * b > w:
                    continue
                cfg = bandred.SevpConfig(n, w, b, getattr(bandred.SevpVariant, var))
                import warnings
                with warnings.catch_warnings():
                    warnings.simplefilter("ignore")
                    r = bandred.reduce_sym_band(A, cfg)
                out[f"{name}_sevp_{w}_{b}_{var}"] = np.array([r.flops["total"]])
            r = bandred.reduce_tri_band(A, w, b)
            out[f"{name}_tri_{w}_{b}"] = np.array([r.flops["total"]])
            for var in ("REFERENCE", "SIMULTANEOUS"):
                cfg = bandred.SvdConfig(n, n, w, b, variant=getattr(bandred.SvdVariant, var))
                r = bandred.reduce_band_svd(A, cfg)
                out[f"{name}_band_{w}_{b}_{var}"] = np.array([r.flops["total"]])
    np.savez_compressed(os.path.join(OUT, "tau0_flops.npz"), **out)
    print(f"wrote {len(out)} arrays")


if __name__ == "__main__":
    main()
