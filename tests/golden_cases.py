"""Loaders for the committed reference golden vectors (tests/golden/*.npz)."""

from __future__ import annotations

import os

import numpy as np

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")

DENSE_CASES = ("scalar", "direct_route", "dense_dual", "cfg1_reduced", "ramp", "decay",
               "r0", "frac_epochs", "epochs_zero", "single_pass", "diverge",
               "diverge_late")


SG_CASES = ("sg_dense", "sg_ramp_r3", "sg_decay", "sg_diverge")


def operator_digest(op) -> str:
    """sha256 over a CSR operator's per-block arrays (relative rowptr, int32
    columns, values): the full-run goldens record the exact operator bits."""
    import hashlib

    h = hashlib.sha256()
    for i in range(1, op.n_blocks + 1):
        ip, ix, d, _ = op.csr_block(i)
        h.update(np.ascontiguousarray(ip - ip[0], dtype=np.int64).tobytes())
        h.update(np.ascontiguousarray(ix[ip[0]:ip[-1]], dtype=np.int32).tobytes())
        h.update(np.ascontiguousarray(d[ip[0]:ip[-1]]).tobytes())
    return h.hexdigest()


def load(name):
    return np.load(os.path.join(GOLDEN, name), allow_pickle=False)


def cfg1_reduced_matrix():
    """Regenerate the cfg1_reduced operator (recipe in make_golden.py)."""
    g = np.random.Generator(np.random.Philox(key=1912))
    a = g.standard_normal((4000, 400)) / np.sqrt(1000.0)
    xt = g.standard_normal(400)
    clean = a @ xt
    eps = g.standard_normal(4000)
    eps *= 0.01 * np.linalg.norm(clean) / np.linalg.norm(eps)
    return a, clean + eps, xt


def dense_case(name):
    d = load("sg_runs.npz" if name.startswith("sg_") else "dense_runs.npz")
    p = name + "/"
    case = {k[len(p):]: d[k] for k in d.files if k.startswith(p)}
    if name == "cfg1_reduced":
        a, b, _ = cfg1_reduced_matrix()
        s = case["A_sum"]
        assert np.isclose(a.sum(), s[0], rtol=0, atol=1e-9) and a[17, 33] == s[2]
        case["A"] = a
    case["refs"] = {k[4:]: v for k, v in case.items() if k.startswith("ref/")}
    case["rel"] = {k[4:]: v for k, v in case.items() if k.startswith("rel/")}
    return case


def case_alphas(case):
    """alpha_k sequence the reference used, from the recorded schedule."""
    from oracle.slimls_oracle import schedule_alpha

    kind = str(case["sched_kind"])
    alpha = float(case["sched_alpha"])
    ramp = int(case["sched_ramp"])
    r = int(case["r"])
    ramp = (r + 1) if (kind == "ramp" and ramp < 0) else (None if ramp < 0 else ramp)
    decay = float(case["sched_decay"])
    k = len(case["indices"])
    return np.array([schedule_alpha(kind, alpha, j, ramp, decay) for j in range(1, k + 1)])


def csr_blocks(d, prefix):
    nb = int(d[f"{prefix}/n_blocks"])
    out = []
    for i in range(nb):
        out.append((d[f"{prefix}/{i}/indptr"], d[f"{prefix}/{i}/indices"],
                    d[f"{prefix}/{i}/data"], tuple(int(v) for v in d[f"{prefix}/{i}/shape"])))
    return out


def tomo_case(name):
    d = load("tomo_runs.npz")
    p = name + "/"
    case = {k[len(p):]: d[k] for k in d.files if k.startswith(p) and "/blocks/" not in k[len(p) - 1:]}
    case["blocks"] = csr_blocks(d, f"{name}/blocks")
    case["rel"] = {k[4:]: v for k, v in case.items() if k.startswith("rel/")}
    return case
