"""Generate the committed golden fixtures from the REFERENCE codec.

Run in the build container (needs /root/reference and oracle/_ref):
    make -C oracle ref && python tests/golden/make_golden.py

Every expected output below comes from oracle/_ref/libhcmx_ref.so, i.e. the
unmodified /root/reference/proj/src/codec.cpp, plus the restated APLR /
matvec glue in oracle/ref_shim.cpp (which calls only reference codec code).
Inputs are seeded; the fixtures let the GPU box (no /root/reference there)
check the oracle and the CUDA path against the reference's own bytes.
"""
from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, os.path.join(ROOT, "oracle"))
sys.path.insert(0, ROOT)

from oracle import Oracle, RefOracle  # noqa: E402

EPS = [0.4, 1e-2, 4.9e-4, 1e-4, 1e-6, 1e-8, 1e-12, 1e-15, 1e-17]
BIG_EPS = [1e-4, 1e-6, 1e-8]  # config-2 accuracies for the 4096-value blocks


def digest(values: np.ndarray) -> str:
    """sha256 of the FP64 bit patterns (exact pin of decompress output)"""
    import hashlib
    return hashlib.sha256(np.ascontiguousarray(values, np.float64).view(np.uint64).tobytes()).hexdigest()


def codec_inputs():
    """(name, values) cases: config-2 style blocks, spans, zeros, edge magnitudes"""
    o = Oracle()
    rng = np.random.default_rng(2024)
    cases = []
    cases.append(("config2_block", o.config2_values(11, 4096)))
    cases.append(("test_codec_afl_oracle", o.log_uniform_signed(42, 4096, 1.0, 1e4)))
    b = o.log_uniform_signed(7, 512, 1e-3, 1e3)
    b[17] = 0.0
    cases.append(("span_with_zero", b))
    cases.append(("empty", np.zeros(0)))
    cases.append(("single", np.array([3.25])))
    cases.append(("constant", np.full(5, 7.5)))
    cases.append(("mixed_zero_signs", np.array([0.0, -1.25, 1.25, -0.0, 0.0])))
    cases.append(("all_zero", np.zeros(33)))
    cases.append(("neg_zeros", np.array([-0.0] * 40)))
    cases.append(("ragged_31", rng.standard_normal(31)))
    cases.append(("ragged_33", rng.standard_normal(33)))
    cases.append(("ragged_1000", rng.standard_normal(1000) * 1e3))
    cases.append(("span_2_127", np.array([1.0, 2.0 ** 127])))
    cases.append(("span_1_128", np.array([1.0, 128.0])))
    cases.append(("huge_span", np.sign(rng.standard_normal(777)) * 10 ** rng.uniform(-300, 300, 777)))
    cases.append(("tiny", np.array([5e-324, 1e-310, 2.2e-308, 1.0])))
    cases.append(("max", np.array([1.7976931348623157e308, 1.0, -1e300])))
    cases.append(("powers2", 2.0 ** np.arange(-20, 21)))
    return cases


def main():
    o, r = Oracle(), RefOracle()
    out = {}
    cases = codec_inputs()
    rec_vals, rec_meta, rec_pay, rec_dec = [], [], [], []
    for ci, (name, v) in enumerate(cases):
        rec_vals.append(v)
        for eps in (EPS if len(v) <= 1024 else BIG_EPS):
            for s in range(4):
                buf = r.compress(v, eps, s)
                dec = r.decompress(buf)
                rec_meta.append((ci, eps, s, buf.e, buf.m, buf.scale, len(buf.payload)))
                rec_pay.append(np.frombuffer(buf.payload, np.uint8))
                rec_dec.append(digest(dec))
    out["case_names"] = np.array([c[0] for c in cases])
    out["case_len"] = np.array([len(v) for v in rec_vals], np.int64)
    out["case_values"] = np.concatenate(rec_vals)
    meta = np.array(rec_meta, dtype=[("case", "<i8"), ("eps", "<f8"), ("scheme", "<i8"),
                                     ("e", "<i8"), ("m", "<i8"), ("scale", "<f8"), ("plen", "<i8")])
    out["meta"] = meta
    out["payload"] = np.concatenate(rec_pay) if rec_pay else np.zeros(0, np.uint8)
    out["decoded_sha256"] = np.array(rec_dec)
    # scalar anchors (test_codec.cpp:25-60)
    eps_list = np.array([4.9e-4, 6.0e-8, 0.5, 1e-300, 1e-4, 1e-6, 1e-8, 0.35, 1e-12, 2 ** -53, 1e-17])
    out["mbits_eps"] = eps_list
    out["mbits"] = np.array([r.mantissa_bits_for(e) for e in eps_list], np.int64)
    stats = np.array([(1.0, 1.0, 0), (1.0, 2.0 ** 127, 0), (1.0, 128.0, 0), (0.0, 0.0, 1),
                      (1.0, 32.0, 0), (1e-6, 1.0, 0), (1.0, 2.0 ** 62, 0), (1.0, 2.0 ** 1022, 0),
                      (5e-324, 1.7e308, 0), (1.0, 2.0 ** 14, 0), (1.0, 2.0 ** 6, 0)])
    out["ebits_stats"] = stats
    out["ebits"] = np.array([r.exponent_bits_for_stats(a, b, int(c)) for a, b, c in stats], np.int64)
    # APLR on given factors (mixedprec.cpp:155-187 glue over the reference codec)
    rng = np.random.default_rng(99)
    ap_meta, ap_pay, ap_in = [], [], []
    for t, (rows, cols, k, eps, s) in enumerate([(48, 40, 3, 1e-8, 0), (64, 64, 8, 1e-6, 0),
                                                 (128, 128, 14, 1e-4, 1), (40, 32, 6, 1e-6, 2),
                                                 (64, 56, 10, 1e-5, 3), (96, 80, 5, 1e-8, 0)]):
        W, _ = np.linalg.qr(rng.standard_normal((rows, k)))
        X, _ = np.linalg.qr(rng.standard_normal((cols, k)))
        sig = 10.0 ** (-0.5 * np.arange(k)) if t != 0 else np.array([1.0, 1e-2, 1e-3])
        bufs = r.aplr_compress(W, X, sig, eps, s)
        ap_in.append((W.ravel(order="F"), X.ravel(order="F"), sig))
        for b in bufs:
            ap_meta.append((t, b.e, b.m, b.scale, len(b.payload)))
            ap_pay.append(np.frombuffer(b.payload, np.uint8))
        out[f"aplr{t}_cfg"] = np.array([rows, cols, k, s], np.int64)
        out[f"aplr{t}_eps"] = np.array([eps])
        out[f"aplr{t}_W"] = ap_in[-1][0]
        out[f"aplr{t}_X"] = ap_in[-1][1]
        out[f"aplr{t}_sigma"] = sig
    out["aplr_meta"] = np.array(ap_meta, dtype=[("case", "<i8"), ("e", "<i8"), ("m", "<i8"),
                                                ("scale", "<f8"), ("plen", "<i8")])
    out["aplr_payload"] = np.concatenate(ap_pay)
    np.savez_compressed(os.path.join(HERE, "codec_golden.npz"), **out)

    # small H-matrix: reference-compressed leaves + reference-glue matvec
    sys.path.insert(0, os.path.dirname(HERE))
    from cpu_hmatrix import build_small_flat  # noqa: E402
    flat, x = build_small_flat(n=768, eps=1e-6, scheme=0, use_ref=True)
    y = r.hmat_matvec(flat, 1.0, x, 0.0, np.zeros(flat.n_rows), threads=1)
    y2 = r.hmat_matvec(flat, -0.5, x, 2.0, y, threads=1)
    np.savez_compressed(os.path.join(HERE, "hmat_golden.npz"), x=x, y=y, y2=y2,
                        **{k: v for k, v in flat.arrays().items()})
    print("wrote", os.listdir(HERE))


if __name__ == "__main__":
    main()
