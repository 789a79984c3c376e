"""Load tests/golden fixtures (written by tests/golden/make_golden.py)."""
from __future__ import annotations

import json
import os

import numpy as np

from oracle_abi import Cfg, Params

HERE = os.path.dirname(os.path.abspath(__file__))
GOLDEN = os.path.join(HERE, "golden", "golden_small.npz")
CONFIGS = os.path.join(HERE, "golden", "golden_configs.json")

_npz = None


def _load():
    global _npz
    if _npz is None:
        _npz = np.load(GOLDEN)
    return _npz


def cases():
    """[(entry, params, kwargs, expected_out)] for every golden case."""
    z = _load()
    index = json.loads(bytes(z["index"]).decode())
    out = []
    for e in index:
        kw = {}
        for k, v in e["scalars"].items():
            kw[k] = Cfg(**v["__cfg__"]) if isinstance(v, dict) and "__cfg__" in v else v
        for k in e["arrays"]:
            kw[k] = z[f"{e['name']}/in/{k}"]
        params = Params(**e["params"]) if e["params"] else None
        out.append((e, params, kw, z[f"{e['name']}/out"]))
    return out


def config_digests():
    with open(CONFIGS) as f:
        return json.load(f)


def run_case(lib, api, params, kw):
    """Replay one golden case through an oracle library (oracle_abi.OracleLib)."""
    if api == "op":
        return lib.op(params, kw["op"], kw["a"], kw["la"], b=kw.get("b"), lb=kw.get("lb", 0), c=kw.get("c", 0.0),
                      vec=kw.get("vec"), k=kw.get("k", 0), n_valid=kw.get("n_valid", 0))
    if api == "fit":
        rc, out = lib.fit(kw["kind"], kw["S"], kw["degree"], kw["lo"], kw["hi"])
        return rc, out, (0,), (0,) * 5
    if api == "eval_encrypted":
        return lib.eval_encrypted(params, kw["coeffs"], kw["lo"], kw["hi"], kw["x"], kw["lx"])
    if api == "newton_refine":
        return lib.newton_refine(params, kw["x"], kw["lx"], kw["y0"], kw["ly"], kw["n"], kw["iters"], kw["n_valid"])
    if api == "invroot":
        return lib.invroot(params, kw["which"], kw["x"], kw["lx"], kw["S"], kw["cfg"], kw["n_valid"])
    if api == "crypto_sign":
        return lib.crypto_sign(params, kw["x"], kw["lx"], kw["mode"], kw["folds"], kw["polys"])
    if api == "stat":
        return lib.stat(params, kw["which"], kw["x"], kw["B"], y=kw.get("y"), cfg=kw.get("cfg"))
    raise ValueError(api)
