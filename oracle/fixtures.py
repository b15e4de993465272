"""Loader for fixture directories written by ``oracle/_ref/bipm_ref dump``.

TEST INFRASTRUCTURE (oracle/): used by tests/ and the fixture scripts only.
Arrays keep the reference layout: a reference ``Matrix(nnz, N)`` (column-major,
one column per scenario, ``proj/core/include/blockipm/types.hpp:56-78``) loads
as a numpy array of shape ``(N, nnz)``, so ``a[b]`` is scenario b's values.
"""
from __future__ import annotations

import json
import os

import numpy as np
import scipy.sparse as sp


class Fixture(dict):
    """dict of arrays plus ``meta`` (the manifest's scalars)."""

    meta: dict

    def csr(self, name: str, values: np.ndarray | None = None) -> sp.csr_matrix:
        """CSR matrix of a shared pattern ``name`` with the given values."""
        rp = self[name + "_rowptr"]
        ci = self[name + "_colind"]
        shape = tuple(self.meta[name + "_shape"])
        if values is None:
            values = self[name + "_val"] if (name + "_val") in self else np.ones(len(ci))
        return sp.csr_matrix((np.asarray(values, dtype=np.float64), ci, rp), shape=shape)

    @property
    def dims(self):
        N, n_x, n_u, m, n_b = self.meta["dims"]
        return N, n_x, n_u, m, n_b


def load_dump(path: str) -> Fixture:
    with open(os.path.join(path, "manifest.json")) as f:
        man = json.load(f)
    fx = Fixture()
    fx.meta = {}
    for k, v in man.items():
        if isinstance(v, dict) and "dtype" in v:
            arr = np.fromfile(os.path.join(path, k + ".bin"), dtype="<" + v["dtype"])
            fx[k] = arr.reshape(v["shape"]) if len(v["shape"]) > 1 else arr
        else:
            fx.meta[k] = v
    return fx


def save_npz(fx: Fixture, path: str) -> None:
    arrays = {k: v for k, v in fx.items()}
    arrays["__meta__"] = np.frombuffer(json.dumps(fx.meta).encode(), dtype=np.uint8)
    np.savez_compressed(path, **arrays)


def load_npz(path: str) -> Fixture:
    z = np.load(path)
    fx = Fixture()
    fx.meta = json.loads(bytes(z["__meta__"]).decode())
    for k in z.files:
        if k != "__meta__":
            fx[k] = z[k]
    return fx
