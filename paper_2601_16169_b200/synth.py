"""Inputs of the sigma path: integral tables, FCIDUMP / determinant-list I/O,
and the deterministic synthetic generator of SURVEY.md 8(d).

Host plumbing only (the reference keeps this host-side too:
integrals.cpp:120-211, detfile.cpp:53-138).

Synthetic generator (configs C1-C5 of BASELINE.json):
  integrals, SplitMix64(seed 2), every 8-fold canonical quadruple set:
    h_pp = -2 + 0.1 p,  h_pq = 0.1 U(-1,1) / (1 + |p-q|)
    (pp|qq) = 0.5 / (1 + |p-q|)
    other (pq|rs) = 0.05 U(-1,1) / (1 + |p-q| + |r-s|),  core = 0
  strings (alpha list = beta list): the aufbau string, then all single,
  double, ... excitations of it in ascending excitation level (each level
  sorted ascending); the last level needed is a SplitMix64(seed 1) random
  subset (partial Fisher-Yates); finally sorted ascending (select_basis,
  oracle.cpp:209-210).
"""
from __future__ import annotations

import itertools
import re
from dataclasses import dataclass
from typing import List, Tuple

import numpy as np

from .errors import FormatError, InputError

GOLDEN = np.uint64(0x9E3779B97F4A7C15)
M64 = (1 << 64) - 1


@dataclass
class Integrals:
    norbs: int
    nelec: int
    ms2: int
    core: float
    h1: np.ndarray   # (n, n)
    eri: np.ndarray  # (n, n, n, n) chemist (pq|rs)


# Configs of BASELINE.json (name -> norbs, total electrons, strings/channel).
CONFIGS = {
    "C1": (16, 10, 1000),
    "C2": (26, 14, 10000),
    "C3": (36, 30, 17320),
    "C4": (36, 54, 31623),
    "C5": (36, 30, 17320),
}


def splitmix64_stream(seed: int, count: int, start: int = 0) -> np.ndarray:
    """Outputs start+1 .. start+count of SplitMix64(seed) (detfile.hpp:38-49)."""
    k = np.arange(start + 1, start + count + 1, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = np.uint64(seed) + k * GOLDEN
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        z = z ^ (z >> np.uint64(31))
    return z


class SplitMix64:
    def __init__(self, seed: int):
        self.state = seed & M64

    def next(self) -> int:
        self.state = (self.state + 0x9E3779B97F4A7C15) & M64
        z = self.state
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & M64
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & M64
        return z ^ (z >> 31)


def uniform_pm1(z: np.ndarray) -> np.ndarray:
    """U[-1, 1] as test_helpers.hpp:51-57."""
    return 2.0 * ((z >> np.uint64(11)).astype(np.float64) / 9007199254740992.0) - 1.0


def random_vector(n: int, seed: int) -> np.ndarray:
    """test::random_vector (test_helpers.hpp:51-57)."""
    return uniform_pm1(splitmix64_stream(seed, n))


def canonical_quadruples(n: int) -> np.ndarray:
    """All 8-fold canonical (p,q,r,s): p>=q, r>=s, (p,q)>=(r,s), lexicographic."""
    p, q, r, s = np.indices((n, n, n, n)).reshape(4, -1)
    keep = (q <= p) & (s <= r) & ((r < p) | ((r == p) & (s <= q)))
    return np.stack([p[keep], q[keep], r[keep], s[keep]], axis=1)


def symmetric_fill(n: int, quads: np.ndarray, vals: np.ndarray) -> np.ndarray:
    eri = np.zeros((n, n, n, n))
    p, q, r, s = quads.T
    for a, b, c, d in ((p, q, r, s), (q, p, r, s), (p, q, s, r), (q, p, s, r),
                       (r, s, p, q), (s, r, p, q), (r, s, q, p), (s, r, q, p)):
        eri[a, b, c, d] = vals
    return eri


def synthetic_integrals(norbs: int, nelec: int, ms2: int = 0, seed: int = 2) -> Integrals:
    n = norbs
    h1 = np.zeros((n, n))
    lower = [(p, q) for p in range(n) for q in range(p)]
    draws = uniform_pm1(splitmix64_stream(seed, len(lower)))
    for (p, q), u in zip(lower, draws):
        h1[p, q] = h1[q, p] = 0.1 * u / (1 + abs(p - q))
    for p in range(n):
        h1[p, p] = -2.0 + 0.1 * p
    quads = canonical_quadruples(n)
    p, q, r, s = quads.T
    coulomb = (p == q) & (r == s)
    vals = np.empty(len(quads))
    vals[coulomb] = 0.5 / (1 + np.abs(p[coulomb] - r[coulomb]))
    nd = int((~coulomb).sum())
    u = uniform_pm1(splitmix64_stream(seed, nd, start=len(lower)))
    vals[~coulomb] = 0.05 * u / (1 + np.abs(p[~coulomb] - q[~coulomb]) + np.abs(r[~coulomb] - s[~coulomb]))
    return Integrals(n, nelec, ms2, 0.0, h1, symmetric_fill(n, quads, vals))


def excitation_level_strings(norbs: int, nel: int, level: int) -> np.ndarray:
    occ = list(range(nel))
    vir = list(range(nel, norbs))
    ref = (1 << nel) - 1
    out = []
    for rem in itertools.combinations(occ, level):
        rm = sum(1 << i for i in rem)
        for add in itertools.combinations(vir, level):
            out.append((ref & ~rm) | sum(1 << a for a in add))
    return np.sort(np.array(out, dtype=np.uint64))


def synthetic_strings(norbs: int, nel: int, count: int, seed: int = 1) -> np.ndarray:
    """Aufbau-near string list of `count` strings (ascending)."""
    chosen: List[np.ndarray] = []
    have = 0
    level = 0
    while have < count:
        lv = excitation_level_strings(norbs, nel, level)
        if len(lv) == 0:
            raise InputError(f"synthetic_strings: only {have} strings exist for {norbs} orbitals / {nel} e")
        need = count - have
        if len(lv) <= need:
            chosen.append(lv)
            have += len(lv)
        else:
            rng = SplitMix64(seed)
            arr = lv.copy()
            for i in range(need):
                j = i + rng.next() % (len(arr) - i)
                arr[i], arr[j] = arr[j], arr[i]
            chosen.append(arr[:need])
            have += need
        level += 1
    return np.sort(np.concatenate(chosen))


def synthetic_system(name: str) -> Tuple[Integrals, np.ndarray, np.ndarray]:
    norbs, nelec, nstr = CONFIGS[name]
    ints = synthetic_integrals(norbs, nelec)
    s = synthetic_strings(norbs, nelec // 2, nstr)
    return ints, s, s.copy()


# ---- FCIDUMP (integrals.cpp:120-211) ---------------------------------------

def parse_fcidump(text: str) -> Integrals:
    lines = text.splitlines()
    header = []
    body_start = None
    for i, line in enumerate(lines):
        up = line.upper()
        cut = [x for x in (up.find("&END"), up.find("/")) if x >= 0]
        if cut:
            header.append(up[: min(cut)])
            body_start = i + 1
            break
        header.append(up)
    if body_start is None:
        raise FormatError("FCIDUMP: unterminated namelist header")
    hdr = " ".join(header)

    def field(name, default=None):
        m = re.search(name + r"[\s=]*([+-]?\d+)", hdr)
        if not m:
            if default is None:
                raise FormatError(f"FCIDUMP: missing or invalid {name}")
            return default
        return int(m.group(1))

    norb, nelec, ms2 = field("NORB"), field("NELEC"), field("MS2", 0)
    if norb <= 0:
        raise FormatError("FCIDUMP: missing or invalid NORB")
    h1 = np.zeros((norb, norb))
    eri = np.zeros((norb,) * 4)
    core = 0.0
    for ln, line in enumerate(lines[body_start:], 1):
        tok = line.split()
        if not tok:
            continue
        try:
            v = float(tok[0].replace("D", "e").replace("d", "e"))
        except ValueError:
            raise FormatError(f"FCIDUMP: non-numeric value '{tok[0]}' on data line {ln}") from None
        if len(tok) != 5:
            raise FormatError(f"FCIDUMP: expected four indices on data line {ln}")
        i, j, k, l = (int(t) for t in tok[1:])
        if min(i, j, k, l) < 0 or max(i, j, k, l) > norb:
            raise FormatError(f"FCIDUMP: index exceeds NORB on data line {ln}")
        if i == j == k == l == 0:
            core = v
        elif k == 0 and l == 0:
            h1[i - 1, j - 1] = h1[j - 1, i - 1] = v
        else:
            p, q, r, s = i - 1, j - 1, k - 1, l - 1
            for a, b, c, d in ((p, q, r, s), (q, p, r, s), (p, q, s, r), (q, p, s, r),
                               (r, s, p, q), (s, r, p, q), (r, s, q, p), (s, r, q, p)):
                eri[a, b, c, d] = v
    return Integrals(norb, nelec, ms2, core, h1, eri)


def write_fcidump(ints: Integrals) -> str:
    out = [f"&FCI NORB={ints.norbs},NELEC={ints.nelec},MS2={ints.ms2},", "&END"]
    quads = canonical_quadruples(ints.norbs)
    # write_fcidump sorts by the packed canonical key p<<48|q<<32|r<<16|s
    for p, q, r, s in quads:
        out.append(f"{ints.eri[p, q, r, s]:.17g} {p + 1} {q + 1} {r + 1} {s + 1}")
    for p in range(ints.norbs):
        for q in range(p + 1):
            if ints.h1[p, q] != 0.0:
                out.append(f"{ints.h1[p, q]:.17g} {p + 1} {q + 1} 0 0")
    out.append(f"{ints.core:.17g} 0 0 0 0")
    return "\n".join(out) + "\n"


# ---- determinant lists (detfile.cpp:53-130) --------------------------------

def write_det_list(norbs: int, alpha, beta) -> str:
    lines = [f"norbs {norbs}", "alpha"] + [f"0x{int(m):x}" for m in alpha] + ["beta"] + [f"0x{int(m):x}" for m in beta]
    return "\n".join(lines) + "\n"


def parse_det_list(text: str):
    norbs = 0
    sec = None
    alpha, beta = [], []
    for ln, line in enumerate(text.splitlines(), 1):
        tok = line.split()
        if not tok or tok[0].startswith("#"):
            continue
        if tok[0] == "norbs":
            norbs = int(tok[1])
            continue
        if tok[0] in ("alpha", "beta"):
            sec = tok[0]
            continue
        if norbs == 0:
            raise FormatError(f"det list: mask before norbs header on line {ln}")
        if sec is None:
            raise FormatError(f"det list: mask outside alpha/beta section on line {ln}")
        m = int(tok[0], 16)
        if m >> norbs:
            raise FormatError(f"det list: mask '{tok[0]}' on line {ln} sets a bit beyond norbs {norbs}")
        (alpha if sec == "alpha" else beta).append(m)
    if norbs == 0:
        raise FormatError("det list: missing norbs header")
    for name, lst in (("alpha", alpha), ("beta", beta)):
        if not lst:
            raise FormatError(f"det list: empty {name} section")
        if len(set(lst)) != len(lst):
            raise FormatError(f"det list: duplicate mask in {name} section")
        if len({bin(m).count('1') for m in lst}) != 1:
            raise FormatError(f"det list: inconsistent electron count in {name} section")
    return norbs, np.array(alpha, dtype=np.uint64), np.array(beta, dtype=np.uint64)


def full_channel_strings(norbs: int, nel: int) -> np.ndarray:
    """All C(norbs, nel) strings ascending (oracle.cpp:214-244)."""
    out = [sum(1 << i for i in c) for c in itertools.combinations(range(norbs), nel)]
    return np.sort(np.array(out, dtype=np.uint64))


def channel_electron_counts(nelec: int, ms2: int) -> Tuple[int, int]:
    na = (nelec + ms2) // 2
    nb = nelec - na
    if (nelec + ms2) % 2 or na < 0 or nb < 0:
        raise InputError(f"inconsistent NELEC {nelec} / MS2 {ms2}")
    return na, nb
