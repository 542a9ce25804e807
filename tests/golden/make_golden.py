"""Generate the committed golden fixtures from the REFERENCE library.

Run in the build container (where /root/reference exists and oracle/_ref is
built):  python tests/golden/make_golden.py

Every expected output below is produced by the unmodified reference
(oracle/_ref/libsemikern_ref.so, compiled from /root/reference/proj/src),
except where the reference has no such function (clip, sparse-Y epilogue):
there the C restatement (oracle/_build/libsk_oracle.so) produces it, and this
script first pins that restatement against the reference on the same inputs
(dense route with the clip inactive, and mxm(CsrMatrix,CsrMatrix) + epilogue).
Inputs are regenerated from seeds; only seeds, small inputs and outputs are
stored.
"""
from __future__ import annotations

import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from oracle.oracle import Port, Ref, RefError  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))


def csr_dict(prefix, a):
    return {f"{prefix}_rows": np.uint32(a.rows), f"{prefix}_cols": np.uint32(a.cols),
            f"{prefix}_rp": a.row_ptr, f"{prefix}_ci": a.col_idx, f"{prefix}_v": a.values}


def epilogue_np(acc, b, clip):
    z = (acc + b).astype(np.float32)
    z = np.where(z < 0, np.float32(0), z)
    if clip > 0:
        z = np.where(z > clip, np.float32(clip), z)
    return z.astype(np.float32)


def main():
    R, P = Ref.get(), Port.get()
    manifest = {}

    # ---- 1. known answers straight from the reference tests ---------------------
    kat = {}
    I2 = R.from_dense(np.eye(2, dtype=np.float32))
    kat["identity_clamp"] = R.relu_forward([I2], [np.zeros(2, np.float32)],
                                           np.array([[3.0], [-2.0]], np.float32)).tolist()
    W = R.from_dense(np.array([[1, 2], [3, 4]], np.float32))
    kat["hand_layer"] = R.relu_forward([W], [np.array([1.0, -100.0], np.float32)],
                                       np.ones((2, 1), np.float32)).tolist()
    A = np.array([[1, 2], [3, 4]], np.float32)
    B = np.array([[5], [6]], np.float32)
    kat["mxm_arith"] = R.mxm_dense_dense(A, B, "arithmetic").tolist()
    kat["mxm_maxplus"] = R.mxm_dense_dense(A, B, "max_plus").tolist()
    kat["all_negative"] = R.dense_relu_forward(
        [R.from_dense(-A)], [np.array([-1, -1], np.float32)],
        np.array([[1, 2], [1, 2]], np.float32)).tolist()
    E3 = R.csr_from_triples(3, 3, [], [], [])
    kat["empty_w"] = R.layer_step(E3, np.zeros(3, np.float32), np.ones((3, 2), np.float32)).tolist()
    I4 = R.from_dense(np.eye(4, dtype=np.float32))
    kat["identity_minus1"] = R.layer_step(I4, np.full(4, -1, np.float32),
                                          np.ones((4, 3), np.float32)).tolist()
    # tuple build cases (test_matrix.cpp:39-88)
    t = R.csr_from_triples(1, 3, [0, 0, 0], [2, 0, 1], [3.0, 1.0, 2.0])
    kat["triples_sorted"] = {"rp": t.row_ptr.tolist(), "ci": t.col_idx.tolist(),
                             "v": t.values.tolist()}
    t = R.csr_from_triples(2, 2, [0, 1], [0, 1], [0.0, 2.0])
    kat["triples_zero_elided"] = {"rp": t.row_ptr.tolist(), "ci": t.col_idx.tolist(),
                                  "v": t.values.tolist()}
    errs = {}
    for name, args in {"out_of_range": (2, 2, [2], [0], [1.0]),
                       "duplicate": (2, 2, [0, 0], [1, 1], [1.0, 2.0]),
                       "dup_after_sort": (3, 3, [2, 0, 2, 1], [1, 0, 1, 2], [1.0, 1.0, 5.0, 0.0]),
                       "first_bad_in_input_order": (4, 4, [0, 9, 5], [0, 1, 0], [1., 1., 1.])}.items():
        try:
            R.csr_from_triples(*args)
            errs[name] = None
        except RefError as e:
            errs[name] = {"kind": e.kind, "msg": str(e).split(": ", 1)[1]}
    kat["triple_errors"] = errs
    verrs = {}
    for name, (rows, cols, rp, ci, v) in {
            "not_monotone": (3, 2, [0, 1, 0, 1], [0], [1.0]),
            "cols_not_increasing": (1, 2, [0, 2], [1, 0], [1.0, 2.0]),
            "col_out_of_range": (1, 2, [0, 1], [5], [1.0]),
            "stored_zero_ok": (1, 2, [0, 2], [0, 1], [0.0, 2.0])}.items():
        from oracle.oracle import csr as mk
        try:
            R.csr_validate(mk(rows, cols, rp, ci, v))
            verrs[name] = None
        except RefError as e:
            verrs[name] = {"kind": e.kind, "msg": str(e).split(": ", 1)[1]}
    kat["validate_errors"] = verrs
    with open(os.path.join(OUT, "kat.json"), "w") as f:
        json.dump(kat, f, indent=1)
    manifest["kat.json"] = "reference"

    # ---- 2. cfg1 full size: the reference's own relu_forward ---------------------
    seed, m, n, L = 42, 1024, 256, 4
    Ws = [P.gen_layer_fixed(m, 16, P.layer_seed(seed, k)) for k in range(L)]
    bs = [np.full(m, -0.05, np.float32) for _ in range(L)]
    y0 = P.gen_input_dense(m, n, seed)
    assert np.array_equal(y0, R.gen_input(m, n, seed)), "gen_input restatement drifted"
    yL = R.relu_forward(Ws, bs, y0, workers=4)
    cat = np.nonzero((yL != 0).any(axis=0))[0].astype(np.uint32)
    np.savez_compressed(os.path.join(OUT, "cfg1.npz"), seed=seed, m=m, n=n, L=L, k=16,
                        bias=np.float32(-0.05), yL=yL, categories=cat,
                        w0_rp=Ws[0].row_ptr, w0_ci=Ws[0].col_idx, w0_v=Ws[0].values)
    manifest["cfg1.npz"] = "reference relu_forward"

    # ---- 3. random models (test_dnn.cpp:153-172 / acceptance.cpp:60-90 style) -----
    rng = np.random.default_rng(101)
    rm = {}
    for trial in range(12):
        mm = int(rng.integers(4, 65))
        layers = int(rng.integers(1, 5))
        nn = int(rng.integers(1, 9))
        inv = float([1, 4, 64][trial % 3])
        s = int(rng.integers(1, 2**62))
        Wt = [R.gen_weight(mm, inv, R.splitmix_at(s, k)) for k in range(layers)]
        bt = [R.gen_bias(mm, R.splitmix_at(s, k), uniform01=bool(trial % 2)) for k in range(layers)]
        yt = R.gen_input(mm, nn, s + 1)
        out = R.relu_forward(Wt, bt, yt)
        dout = R.dense_relu_forward(Wt, bt, yt)
        rm[f"t{trial}_meta"] = np.array([mm, layers, nn], np.int64)
        rm[f"t{trial}_y0"] = yt
        rm[f"t{trial}_out"] = out
        rm[f"t{trial}_dense_out"] = dout
        for k in range(layers):
            rm.update(csr_dict(f"t{trial}_w{k}", Wt[k]))
            rm[f"t{trial}_b{k}"] = bt[k]
    np.savez_compressed(os.path.join(OUT, "random_models.npz"), **rm)
    manifest["random_models.npz"] = "reference relu_forward + dense_relu_forward"

    # ---- 4. cfg2 single layer, reduced batch, two densities ------------------------
    c2 = {}
    m2, n2 = 4096, 64
    y2 = P.gen_input_dense(m2, n2, 7)
    for d in (0.01, 0.001):
        Wd = P.gen_layer_density(m2, d, P.layer_seed(7, 0))
        key = f"d{d:g}".replace(".", "p")
        c2[f"{key}_out"] = R.layer_step(Wd, np.full(m2, -0.05, np.float32), y2, workers=4)
        c2[f"{key}_nnz"] = np.int64(Wd.nnz)
    np.savez_compressed(os.path.join(OUT, "cfg2_small.npz"), m=m2, n=n2, seed=7, **c2)
    manifest["cfg2_small.npz"] = "reference layer_step"

    # ---- 5. cfg3 construction, reduced batch, sparse activations --------------------
    m3, n3, L3, kY = 16384, 96, 3, 246
    W3 = [P.gen_layer_fixed(m3, 32, P.layer_seed(3, k), 1.0 / 16) for k in range(L3)]
    b3 = np.full(m3, -0.3, np.float32)
    Y = P.gen_input_binary(m3, n3, kY, 3)
    # pin the restated sparse layer against the reference on layer 1:
    Z = R.mxm_csr_csr(W3[0], Y, workers=4)
    Zd = Z.to_dense()
    touched = np.zeros_like(Zd, dtype=bool)
    for i in range(Z.rows):
        touched[i, Z.col_idx[Z.row_ptr[i]:Z.row_ptr[i + 1]]] = True
    ref_layer1 = np.where(touched, epilogue_np(Zd, b3[:, None], 32.0), 0).astype(np.float32)
    port_layer1 = P.layer_sparse(W3[0], b3, Y, 32.0).to_dense()
    assert np.array_equal(ref_layer1, port_layer1), "sparse restatement != reference mxm+epilogue"
    trace = [Y.nnz]
    Yk = Y
    for k in range(L3):
        Yk = P.layer_sparse(W3[k], b3, Yk, 32.0)
        trace.append(Yk.nnz)
    np.savez_compressed(os.path.join(OUT, "cfg3_small.npz"), m=m3, n=n3, L=L3, kY=kY, seed=3,
                        trace=np.array(trace, np.int64), **csr_dict("yL", Yk),
                        layer1_nnz=np.int64((port_layer1 != 0).sum()))
    manifest["cfg3_small.npz"] = "restatement, pinned to reference mxm_csr_csr + epilogue"

    with open(os.path.join(OUT, "MANIFEST.json"), "w") as f:
        json.dump(manifest, f, indent=1)
    print("golden fixtures written:", sorted(manifest))


if __name__ == "__main__":
    main()
