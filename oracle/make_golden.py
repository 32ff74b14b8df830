"""TEST INFRASTRUCTURE ONLY -- generate tests/golden/*.npz by running the reference itself.

Runs the reference package (``tilekit`` from oracle/_ref, built by ``make -C oracle ref``
from /root/reference/pkg; or straight from /root/reference/pkg/src) on small seeded cases
and stores inputs, outputs, event counters and resolved tilings.  These fixtures pin both
the oracle restatement (tests/test_oracle.py, bitwise) and the B200 path (tests/).

    python oracle/make_golden.py            # writes tests/golden/
"""

from __future__ import annotations

import dataclasses
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
OUT = os.path.join(os.path.dirname(HERE), "tests", "golden")


def _reference():
    for path in (os.path.join(HERE, "_ref"), "/root/reference/pkg/src"):
        if os.path.isdir(os.path.join(path, "tilekit")):
            sys.path.insert(0, path)
            import tilekit

            return tilekit
    raise SystemExit("reference tilekit not found (run `make -C oracle ref`)")


tk = _reference()


def counters_dict(c):
    return {f.name: int(getattr(c, f.name)) for f in dataclasses.fields(c)}


def save(name, meta, **arrays):
    os.makedirs(OUT, exist_ok=True)
    np.savez_compressed(os.path.join(OUT, f"{name}.npz"), meta=json.dumps(meta), **arrays)


def dense_cases():
    rng = np.random.default_rng(2)
    for trans_a, trans_b in ((False, False), (False, True), (True, False), (True, True)):
        m, n, k = 48, 40, 24
        a = rng.standard_normal((m, k)).astype(np.float32)
        b = rng.standard_normal((k, n)).astype(np.float32)
        c = rng.standard_normal((m, n)).astype(np.float32)
        cfg = tk.build_dense_config(m, n, k, np.float32, trans_a=trans_a, trans_b=trans_b,
                                    operator_shape=(8, 8, 8))
        d = np.zeros(m * n, np.float32)
        a_buf = (a.T if trans_a else a).copy(order="F").ravel(order="F")
        b_buf = (b.T if trans_b else b).copy(order="F").ravel(order="F")
        cnt = tk.matmul(cfg, a_buf, b_buf, c.ravel(order="F"), d)
        res = tk.kernel.resolve_config(cfg)
        tag = ("t" if trans_a else "n") + ("t" if trans_b else "n")
        save(f"dense_f32_{tag}", {"m": m, "n": n, "k": k, "trans_a": trans_a, "trans_b": trans_b,
                                  "block_tile": list(res.params.block_tile),
                                  "counters": counters_dict(cnt)},
             a=a, b=b, c=c, d=d.reshape((m, n), order="F"))
    # fp16-valued inputs at a tensor-core-friendly size (the oracle protocol for half storage)
    m, n, k = 128, 256, 192
    a = rng.standard_normal((m, k)).astype(np.float16).astype(np.float32)
    b = rng.standard_normal((k, n)).astype(np.float16).astype(np.float32)
    c = rng.standard_normal((m, n)).astype(np.float32)
    cfg = tk.build_dense_config(m, n, k, np.float32)
    d = np.zeros(m * n, np.float32)
    cnt = tk.matmul(cfg, a.ravel(order="F"), b.ravel(order="F"), c.ravel(order="F"), d)
    save("dense_f16valued", {"m": m, "n": n, "k": k, "counters": counters_dict(cnt),
                             "block_tile": list(tk.kernel.resolve_config(cfg).params.block_tile)},
         a=a, b=b, c=c, d=d.reshape((m, n), order="F"))
    # f64 and wide accumulation on integers
    m = n = k = 32
    a = rng.integers(-8, 9, (m, k)).astype(np.float64)
    b = rng.integers(-8, 9, (k, n)).astype(np.float64)
    c = rng.integers(-8, 9, (m, n)).astype(np.float64)
    cfg = tk.build_dense_config(m, n, k, np.float64, block_tile=(16, 16, 8))
    d = np.zeros(m * n)
    cnt = tk.matmul(cfg, a.ravel(order="F"), b.ravel(order="F"), c.ravel(order="F"), d)
    save("dense_f64_int", {"m": m, "n": n, "k": k, "block_tile": [16, 16, 8],
                           "counters": counters_dict(cnt)}, a=a, b=b, c=c,
         d=d.reshape((m, n), order="F"))
    m = n = k = 64
    a = rng.standard_normal((m, k)).astype(np.float32)
    b = rng.standard_normal((k, n)).astype(np.float32)
    c = rng.standard_normal((m, n)).astype(np.float32)
    cfg = tk.build_dense_config(m, n, k, np.float32, wide_accumulate=True, block_tile=(32, 32, 8))
    d = np.zeros(m * n, np.float32)
    cnt = tk.matmul(cfg, a.ravel(order="F"), b.ravel(order="F"), c.ravel(order="F"), d)
    save("dense_f32_wide", {"m": m, "n": n, "k": k, "block_tile": [32, 32, 8],
                            "counters": counters_dict(cnt)}, a=a, b=b, c=c,
         d=d.reshape((m, n), order="F"))


def c1_cases():
    """BASELINE configs[0] (C1): fp16-valued 256^3 column-major at the reference's DEFAULT
    tiling (build_dense_config resolves block (256, 256, 8), op (8, 8, 8)), f32 k-ascending."""
    rng = np.random.default_rng(256)
    m = n = k = 256
    a = rng.standard_normal((m, k)).astype(np.float16).astype(np.float32)
    b = rng.standard_normal((k, n)).astype(np.float16).astype(np.float32)
    c = rng.standard_normal((m, n)).astype(np.float32)
    cfg = tk.build_dense_config(m, n, k, np.float32)
    d = np.zeros(m * n, np.float32)
    cnt = tk.matmul(cfg, a.ravel(order="F"), b.ravel(order="F"), c.ravel(order="F"), d)
    res = tk.kernel.resolve_config(cfg)
    save("c1_dense_256", {"m": m, "n": n, "k": k, "counters": counters_dict(cnt),
                          "block_tile": list(res.params.block_tile),
                          "operator_shape": list(res.params.operator_shape)},
         a=a, b=b, c=c, d=d.reshape((m, n), order="F"))


def padded_cases():
    """Padded layouts (reference layouts.py:132-188, builder 414-418): padded SHARED staging
    (build_dense_config(shared_pad=...): the heuristic sees the padded footprint) and padded
    GLOBAL A / B / C / D buffers (physical size (rows + pad) * cols, padding never observed)."""
    from tilekit import layouts as L

    rng = np.random.default_rng(414)
    m, n, k = 128, 192, 96
    a = rng.standard_normal((m, k)).astype(np.float16).astype(np.float32)
    b = rng.standard_normal((k, n)).astype(np.float16).astype(np.float32)
    c = rng.standard_normal((m, n)).astype(np.float32)
    cfg = tk.build_dense_config(m, n, k, np.float32, shared_pad=4)
    d = np.zeros(m * n, np.float32)
    cnt = tk.matmul(cfg, a.ravel(order="F"), b.ravel(order="F"), c.ravel(order="F"), d)
    res = tk.kernel.resolve_config(cfg)
    save("padded_shared", {"m": m, "n": n, "k": k, "pad": 4, "counters": counters_dict(cnt),
                           "block_tile": list(res.params.block_tile)},
         a=a, b=b, c=c, d=d.reshape((m, n), order="F"))
    pads = {"A": 8, "B": 3, "C": 4, "D": 5}
    cfg = dataclasses.replace(
        tk.build_dense_config(m, n, k, np.float32),
        global_a_layout=L.Padded(L.ColMajor(np.float32, ("M", "K"), (m, k)), pads["A"]),
        global_b_layout=L.Padded(L.ColMajor(np.float32, ("K", "N"), (k, n)), pads["B"]),
        global_c_layout=L.Padded(L.ColMajor(np.float32, ("M", "N"), (m, n)), pads["C"]),
        global_d_layout=L.Padded(L.ColMajor(np.float32, ("M", "N"), (m, n)), pads["D"]))

    def pad_buf(x, p):
        buf = np.full((x.shape[0] + p, x.shape[1]), -7.0, np.float32)
        buf[:x.shape[0]] = x
        return buf.ravel(order="F")

    dbuf = np.full((m + pads["D"]) * n, 123.0, np.float32)
    cnt = tk.matmul(cfg, pad_buf(a, pads["A"]), pad_buf(b, pads["B"]), pad_buf(c, pads["C"]), dbuf)
    save("padded_global", {"m": m, "n": n, "k": k, "pads": pads, "counters": counters_dict(cnt)},
         a=a, b=b, c=c, d_buf=dbuf)


def fused_cases():
    rng = np.random.default_rng(12)
    m, n, k = 128, 96, 64
    bias = rng.standard_normal(n).astype(np.float32)
    cfg = tk.build_fused_config(m, n, k, np.float32, bias=bias, relu_on_c=True, relu_on_d=True,
                                add_a=0.5, add_b=-0.25, block_tile=(32, 32, 16))
    a = rng.standard_normal((m, k)).astype(np.float32)
    b = rng.standard_normal((k, n)).astype(np.float32)
    c = rng.standard_normal((m, n)).astype(np.float32)
    d = np.zeros(m * n, np.float32)
    cnt = tk.matmul(cfg, a.ravel(order="F"), b.ravel(order="F"), c.ravel(order="F"), d)
    save("fused_f32", {"m": m, "n": n, "k": k, "block_tile": [32, 32, 16],
                       "relu_on_c": True, "relu_on_d": True, "add_a": 0.5, "add_b": -0.25,
                       "counters": counters_dict(cnt)},
         a=a, b=b, c=c, bias=bias, d=d.reshape((m, n), order="F"))
    # scaling transforms + transposes + bias/relu (SURVEY 8d C3 composition), bias axis m
    m, n, k = 64, 48, 32
    alpha, beta = 1.5, 0.5
    a = rng.standard_normal((k, m)).astype(np.float32)   # stored transposed
    b = rng.standard_normal((k, n)).astype(np.float32)
    c = rng.standard_normal((m, n)).astype(np.float32)
    bias_m = rng.standard_normal(m).astype(np.float32)
    from tilekit.components import BiasEpilogue, relu, scale

    cfg = dataclasses.replace(
        tk.build_dense_config(m, n, k, np.float32, trans_a=True, block_tile=(16, 16, 8)),
        transform_g2s_c=scale(beta / alpha), transform_r2s_d=scale(alpha),
        epilogue=BiasEpilogue(bias_m, axis="m"), transform_s2g_d=relu)
    d = np.zeros(m * n, np.float32)
    cnt = tk.matmul(cfg, a.ravel(order="F"), b.ravel(order="F"), c.ravel(order="F"), d)
    save("scaled_bias_m_relu", {"m": m, "n": n, "k": k, "alpha": alpha, "beta": beta,
                                "block_tile": [16, 16, 8], "counters": counters_dict(cnt)},
         a=a, b=b, c=c, bias=bias_m, d=d.reshape((m, n), order="F"))


def pair_cases():
    rng = np.random.default_rng(6)
    m, n, k = 32, 24, 16
    mk = lambda s: np.asfortranarray((rng.standard_normal(s) + 1j * rng.standard_normal(s))
                                     .astype(np.complex64))
    a, b, c = mk((m, k)), mk((k, n)), mk((m, n))
    c_in = c.copy(order="F")
    tk.gemm_ex(False, False, 1 + 1j, a, b, 2.0, c, operator_shape=(8, 8, 8))
    save("complex_gemm_ex", {"m": m, "n": n, "k": k, "alpha": [1.0, 1.0], "beta": [2.0, 0.0]},
         a=a, b=b, c=c_in, d=c)
    m, n, k = 64, 64, 32
    a, b, c = mk((m, k)), mk((k, n)), mk((m, n))
    cfg = tk.build_complex_config(m, n, k, np.complex64, block_tile=(32, 32, 16))
    d = np.zeros(m * n, np.complex64)
    cnt = tk.matmul(cfg, a.ravel(order="F").view(np.float32), b.ravel(order="F").view(np.float32),
                    c.ravel(order="F").view(np.float32), d.view(np.float32))
    save("complex_matmul", {"m": m, "n": n, "k": k, "block_tile": [32, 32, 16],
                            "counters": counters_dict(cnt)}, a=a, b=b, c=c,
         d=d.reshape((m, n), order="F"))
    for dual_t, name in ((tk.DUAL32, "dual32"), (tk.DUAL64, "dual64")):
        m = n = k = 32
        v = lambda s: rng.standard_normal(s).astype(dual_t["value"])
        a = np.asfortranarray(tk.dual_array(v((m, k)), v((m, k)), dual_t))
        b = np.asfortranarray(tk.dual_array(v((k, n)), v((k, n)), dual_t))
        c = np.asfortranarray(tk.dual_array(v((m, n)), v((m, n)), dual_t))
        cfg = tk.build_dual_config(m, n, k, dual_t, block_tile=(16, 16, 16))
        d = np.zeros(m * n, dual_t)
        sc = dual_t["value"]
        cnt = tk.matmul(cfg, a.ravel(order="F").view(sc), b.ravel(order="F").view(sc),
                        c.ravel(order="F").view(sc), d.view(sc))
        save(f"{name}_matmul", {"m": m, "n": n, "k": k, "block_tile": [16, 16, 16],
                                "counters": counters_dict(cnt)}, a=a, b=b, c=c,
             d=d.reshape((m, n), order="F"))


def variant_cases():
    rng = np.random.default_rng(8)
    n = 64
    cfg = tk.build_diagonal_config(n, np.float32, block_tile=(16, 16, 8))
    diag = rng.standard_normal(n).astype(np.float32)
    b = rng.standard_normal((n, n)).astype(np.float32)
    c = rng.standard_normal((n, n)).astype(np.float32)
    d = np.zeros(n * n, np.float32)
    cnt = tk.matmul(cfg, diag, b.ravel(order="F"), c.ravel(order="F"), d)
    save("diagonal", {"n": n, "block_tile": [16, 16, 8], "counters": counters_dict(cnt)},
         diag=diag, b=b, c=c, d=d.reshape((n, n), order="F"))
    for na, nb, nc, nd in ((2, 4, 8, 8), (8, 4, 16, 16), (16, 8, 32, 32)):
        a = np.asfortranarray(rng.standard_normal((nb, nd, na)).astype(np.float32))
        bb = np.asfortranarray(rng.standard_normal((nd, nc)).astype(np.float32))
        dd, cnt = tk.contract(a, bb)
        res = tk.kernel.resolve_config(tk.build_tc_config(na, nb, nc, nd, np.float32))
        save(f"tc_{na}_{nb}_{nc}_{nd}", {"na": na, "nb": nb, "nc": nc, "nd": nd,
                                         "block_tile": list(res.params.block_tile),
                                         "operator_shape": list(res.params.operator_shape),
                                         "counters": counters_dict(cnt)}, a=a, b=bb, d=dd)
    # alpha = 0: C := beta * C, A/B never read
    m = n = k = 16
    c = np.asfortranarray(rng.standard_normal((m, n)).astype(np.float32))
    c0 = c.copy(order="F")
    cnt = tk.gemm_ex(False, False, 0.0, np.full((m, k), np.nan, np.float32),
                     np.full((k, n), np.inf, np.float32), 3.0, c, operator_shape=(8, 8, 8))
    save("alpha_zero", {"m": m, "n": n, "k": k, "beta": 3.0, "counters": counters_dict(cnt)},
         c=c0, d=c)
    # gemm_ex_raw over raw pointers
    m, n, k = 16, 16, 8
    a = np.asfortranarray(rng.standard_normal((m, k)).astype(np.float32))
    b = np.asfortranarray(rng.standard_normal((k, n)).astype(np.float32))
    c = np.asfortranarray(rng.standard_normal((m, n)).astype(np.float32))
    c0 = c.copy(order="F")
    st = tk.gemm_ex_raw(0, 0, 0, m, n, k, 1.5, 0.0, a.ctypes.data, b.ctypes.data, 0.25, 0.0,
                        c.ctypes.data)
    save("gemm_ex_raw_f32", {"m": m, "n": n, "k": k, "alpha": 1.5, "beta": 0.25, "status": st},
         a=a, b=b, c=c0, d=c)


GETT_CASES = (("abcd-aebf-dfce", dict(a=8, b=4, c=4, d=6, e=4, f=6)),
              ("abc-acd-db", dict(a=8, b=16, c=4, d=8)),
              ("ab-cad-dcb", dict(a=16, b=24, c=2, d=4)),
              # five M digits, four K digits, three N digits, all interleaved (rank-5 maps)
              ("axbyczde-fabgchdie-xhzfigy", dict(a=2, b=4, c=2, d=2, e=2, f=2, g=4, h=2, i=2,
                                                  x=4, y=2, z=4)))


def gett_cases():
    """General contractions through the reference's own StridedPermutation layouts
    (layouts.py:435-506), wired like its build_tc_config (api.py:259-290) but for any
    TCCG spec 'D-A-B': M = A-free indices in D order, N = B-free in D order, K = contracted
    indices in A order."""
    rng = np.random.default_rng(9)
    L = tk.layouts
    for spec, ext in GETT_CASES:
        d_idx, a_idx, b_idx = spec.split("-")
        m_idx = [i for i in d_idx if i in a_idx]
        n_idx = [i for i in d_idx if i in b_idx]
        k_idx = [i for i in a_idx if i in b_idx]
        vol = lambda idx: int(np.prod([ext[i] for i in idx]))
        m, n, k = vol(m_idx), vol(n_idx), vol(k_idx)
        grp = lambda idx: tuple((i, ext[i]) for i in idx)
        dt = np.dtype(np.float32)
        base = tk.build_dense_config(m, n, k, dt, operator_shape=(8, 8, 8))
        cfg = dataclasses.replace(
            base,
            global_a_layout=L.StridedPermutation(dt, ("M", "K"), (m, k), dim_map={"M": grp(m_idx), "K": grp(k_idx)},
                                                 storage_order=tuple(a_idx)),
            global_b_layout=L.StridedPermutation(dt, ("K", "N"), (k, n), dim_map={"K": grp(k_idx), "N": grp(n_idx)},
                                                 storage_order=tuple(b_idx)),
            global_c_layout=L.Zero(dt, ("M", "N"), (m, n)),
            global_d_layout=L.StridedPermutation(dt, ("M", "N"), (m, n), dim_map={"M": grp(m_idx), "N": grp(n_idx)},
                                                 storage_order=tuple(d_idx)))
        a = np.asfortranarray(rng.standard_normal([ext[i] for i in a_idx]).astype(np.float32))
        b = np.asfortranarray(rng.standard_normal([ext[i] for i in b_idx]).astype(np.float32))
        d = np.zeros(m * n, np.float32)
        cnt = tk.matmul(cfg, a.ravel(order="F"), b.ravel(order="F"), np.zeros(0, np.float32), d)
        res = tk.kernel.resolve_config(cfg)
        save("gett_" + spec.replace("-", "_"), {"spec": spec, "sizes": ext,
                                                "block_tile": list(res.params.block_tile),
                                                "counters": counters_dict(cnt)},
             a=a, b=b, d=d.reshape([ext[i] for i in d_idx], order="F"))


def host_logic_cases():
    """Resolved tilings and counters (no element data) for the planner/counter tests."""
    cases = []
    for m, n, k, dtype, budget, block in ((256, 256, 256, "f32", None, None),
                                          (1024, 1024, 1024, "f32", None, None),
                                          (8192, 8192, 8192, "f32", None, None),
                                          (128, 128, 128, "f32", None, (64, 64, 16)),
                                          (512, 256, 64, "f64", None, None),
                                          (256, 512, 128, "f32", 16384, None),
                                          (128, 128, 128, "f32", (128 * 16 + 16 * 128) * 4, None)):
        dt = np.float32 if dtype == "f32" else np.float64
        cfg = tk.build_dense_config(m, n, k, dt, block_tile=block,
                                    operator_shape=(8, 8, 16) if budget == (128 * 16 + 16 * 128) * 4 else None)
        if budget is not None:
            cfg = dataclasses.replace(cfg, params=dataclasses.replace(cfg.params, scratch_budget=budget))
        res = tk.kernel.resolve_config(cfg)
        cases.append({"m": m, "n": n, "k": k, "dtype": dtype, "budget": budget, "block": block,
                      "operator_shape": list(res.params.operator_shape),
                      "resolved_block": list(res.params.block_tile)})
    with open(os.path.join(OUT, "host_logic.json"), "w") as f:
        json.dump({"tilings": cases,
                   "diag_hand_case": __import__("tilekit.bench").bench.expected_diagonal_counters((32, 32, 32), (16, 16, 8))},
                  f, indent=1)


if __name__ == "__main__":
    print("reference lane:", tk.active_lane())
    which = sys.argv[1:] or ["dense", "c1", "padded", "fused", "pair", "variant", "gett", "host_logic"]
    for name in which:
        globals()[f"{name}_cases"]()
    print("wrote", sorted(os.listdir(OUT)))
