"""Test helper: MATPOWER case text -> the reference's CaseData tables.

Column selection follows the reference's row structs (opf.hpp:19-51) and its
reader (opf_parse.cpp:102-214): bus (id type Pd Qd Gs Bs Vm Va Vmax Vmin from
MATPOWER columns 0-5, 7, 8, 11, 12), gen (bus Pg Qg Qmax Qmin Vg status Pmax
Pmin from 0-5, 7-9), branch (from to r x b rateA tap shift status from 0-5,
8-10), gencost (model startup shutdown ncost + coefficients).  Used only to
feed bipm_problem_create_tables in tests; the product never parses here.
"""
import re

import numpy as np


def _table(text: str, name: str):
    m = re.search(r"mpc\." + name + r"\s*=\s*\[(.*?)\]", text, re.S)
    rows = []
    for line in m.group(1).split("\n"):
        line = line.split("%")[0].strip().rstrip(";").strip()
        if line:
            rows.append([float(v) for v in line.replace(";", " ").split()])
    return rows


def read_case(path: str) -> dict:
    text = open(path).read()
    base = float(re.search(r"mpc\.baseMVA\s*=\s*([0-9.eE+-]+)", text).group(1))
    bus = np.array([[r[0], r[1], r[2], r[3], r[4], r[5], r[7], r[8], r[11], r[12]]
                    for r in _table(text, "bus")])
    gen = np.array([[r[0], r[1], r[2], r[3], r[4], r[5], r[7], r[8], r[9]]
                    for r in _table(text, "gen")])
    branch = np.array([[r[0], r[1], r[2], r[3], r[4], r[5], r[8], r[9], r[10]]
                       for r in _table(text, "branch")])
    gc = _table(text, "gencost")
    gencost = np.array([r[:4] for r in gc])
    coef = np.array([c for r in gc for c in r[4:4 + int(r[3])]])
    return dict(base_mva=base, bus=bus, gen=gen, branch=branch, gencost_rows=gencost,
                gencost_coef=coef)


def draw_multipliers(nbus: int, N: int, sigma: float, seed: int) -> np.ndarray:
    """Not the reference's mt19937_64 stream -- any [N][nbus] table works for
    the tables constructor; tests that need the reference's draws take them
    from the problem built from the case file (array 'mult')."""
    rng = np.random.default_rng(seed)
    return np.clip(rng.normal(1.0, sigma, size=(N, nbus)), 0.5, 1.5)
