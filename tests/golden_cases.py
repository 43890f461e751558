"""Load the golden fixtures (made by tests/golden/make_golden.py from the
unmodified reference) and rebuild the matching oracle instance."""

from __future__ import annotations

import json
from functools import lru_cache
from pathlib import Path

import numpy as np

from oracle import hks_oracle as O
from paper_1701_02324_b200 import workloads

GOLDEN = Path(__file__).resolve().parent / "golden"

WORKLOAD_CASES = {"c1_n4096": "C1", "c2_n8192": "C2", "c3_n8192": "C3",
                  "c4_n8192": "C4", "c5_n2048": "C5"}
ALL_CASES = ["tiny_n10", "rank0_n128", "frozen_n1024", "laplace_n1024",
             "poly_n1024", "gauss_uniform_n2000", "c1_n4096", "c2_n8192",
             "c3_n8192", "c4_n8192", "c5_n2048"]


@lru_cache(maxsize=None)
def load(name):
    z = np.load(GOLDEN / f"{name}.npz")
    g = {k: z[k] for k in z.files}
    g["meta"] = json.loads(str(g["meta"]))
    return g


def coords_for(name):
    g = load(name)
    if "coords" in g:
        return g["coords"]
    w = workloads.CONFIGS[WORKLOAD_CASES[name]].scaled(g["meta"]["n"])
    return workloads.points(w, 0)


def kern_of(meta):
    return {"family": meta["family"], "h": meta["h"], "degree": meta["degree"],
            "shift": meta["shift"]}


def rhs_for(meta):
    return np.random.default_rng([meta["seed"], 1000]).standard_normal(
        (meta["n"], meta["nrhs"]))


def matvec_w(meta):
    return np.random.default_rng([meta["seed"], 78]).standard_normal(meta["n"])


def sketch_vec(tag, node, n):
    return np.random.default_rng([tag, node]).standard_normal(n)


@lru_cache(maxsize=None)
def oracle_instance(name, threads=8):
    g = load(name)
    m = g["meta"]
    x = coords_for(name)
    inst = O.pipeline(x, kern_of(m), m["leaf"], m["tau"], m["max_rank"],
                      m["samples"], m["mode"], m["seed"], kappa=m["kappa"],
                      threads=threads)
    inst["fac"] = O.factorize(inst["tree"], inst["skel"], inst["leaf"],
                              inst["coup"], m["lam"], threads=threads)
    inst["coords_in"] = x
    return inst


def skel_list(g, i):
    return g["skel_idx"][g["skel_off"][i]:g["skel_off"][i + 1]]
