"""Test helpers: golden loaders and matrix builders (tests only)."""
import json
import os

import numpy as np

import paper_1003_0952_b200 as P

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def known_answers():
    with open(os.path.join(GOLDEN, "known_answers.json")) as f:
        return json.load(f)


def matrix_from_dict(d):
    vs = bool(d.get("value_symmetric", False))
    return P.CsrcMatrix(int(d["n"]), np.asarray(d["ad"], np.float64), np.asarray(d["ia"], np.int32),
                        np.asarray(d["ja"], np.int32), np.asarray(d["al"], np.float64),
                        np.asarray(d["au"] if not vs else [], np.float64), vs)


class Golden:
    """Lazy view of tests/golden/<name>.npz."""

    def __init__(self, name):
        self.z = np.load(os.path.join(GOLDEN, name), allow_pickle=False)
        self.names = [str(s) for s in self.z["names"]]

    def has(self, key):
        return key in self.z.files

    def __getitem__(self, key):
        return self.z[key]

    def matrix(self, prefix):
        z = self.z
        vs = bool(int(z[prefix + "vs"])) if prefix + "vs" in z.files else False
        n = int(z[prefix + "ia"].size - 1)
        return P.CsrcMatrix(n, z[prefix + "ad"], z[prefix + "ia"], z[prefix + "ja"], z[prefix + "al"],
                            z[prefix + "au"] if not vs else np.zeros(0), vs)


def family():
    return Golden("family.npz")


def meshes():
    return Golden("meshes.npz")


def rel_l2(y, ref):
    ref = np.asarray(ref, np.float64)
    nrm = np.linalg.norm(ref)
    d = np.linalg.norm(np.asarray(y, np.float64) - ref)
    return d / nrm if nrm > 0 else d


def rel_inf(y, ref):
    """relative_error (bench.hpp:93-100)."""
    ref = np.asarray(ref, np.float64)
    if ref.size == 0:
        return 0.0
    num = np.max(np.abs(np.asarray(y, np.float64) - ref))
    den = np.max(np.abs(ref))
    return num if den == 0.0 else num / den


def round32(a):
    """fp32-rounded copy of a CSRC matrix (fp64 oracle on fp32 inputs)."""
    return P.CsrcMatrix(a.n, a.ad.astype(np.float32).astype(np.float64), a.ia, a.ja,
                        a.al.astype(np.float32).astype(np.float64),
                        a.au.astype(np.float32).astype(np.float64), a.value_symmetric)
