"""Input plumbing: synthetic generator of SURVEY.md 8(d), FCIDUMP and
determinant-list I/O (integrals.cpp:120-211, detfile.cpp:53-138).  CPU only."""
import numpy as np
import pytest

from paper_2601_16169_b200 import errors, synth
from util import FIXTURES, GOLDEN, golden_meta, load_fixture


def test_splitmix_stream_matches_sequential():
    rng = synth.SplitMix64(7)
    seq = np.array([rng.next() for _ in range(100)], dtype=np.uint64)
    assert np.array_equal(seq, synth.splitmix64_stream(7, 100))
    v = synth.random_vector(1000, 3)
    assert v.min() >= -1.0 and v.max() <= 1.0


@pytest.mark.parametrize("name", FIXTURES)
def test_fcidump_parser_matches_reference_parse(name):
    ints, d = load_fixture(name)            # dense arrays from the reference parse_fcidump
    mine = synth.parse_fcidump((GOLDEN / "fixtures" / f"{name}.fcidump").read_text())
    assert (mine.norbs, mine.nelec, mine.ms2) == (ints.norbs, ints.nelec, ints.ms2)
    assert mine.core == ints.core
    assert np.array_equal(mine.h1, ints.h1) and np.array_equal(mine.eri, ints.eri)


def test_fcidump_round_trip_is_exact():
    ints = synth.synthetic_integrals(7, 4)
    back = synth.parse_fcidump(synth.write_fcidump(ints))
    assert np.array_equal(back.h1, ints.h1) and np.array_equal(back.eri, ints.eri)


def test_fcidump_errors():
    with pytest.raises(errors.FormatError):
        synth.parse_fcidump("&FCI NORB=2,NELEC=2\n1.0 1 1 1 1\n")           # no &END
    with pytest.raises(errors.FormatError):
        synth.parse_fcidump("&FCI NELEC=2,&END\n")
    with pytest.raises(errors.FormatError):
        synth.parse_fcidump("&FCI NORB=2,NELEC=2,&END\n1.0 1 1 3 1\n")      # index > NORB
    with pytest.raises(errors.FormatError):
        synth.parse_fcidump("&FCI NORB=2,NELEC=2,&END\nabc 1 1 1 1\n")
    ok = synth.parse_fcidump("&FCI NORB=2,NELEC=2,&END\n1.5D-1 1 2 0 0\n")
    assert ok.h1[0, 1] == ok.h1[1, 0] == 0.15


def test_det_list_round_trip_and_errors():
    a = synth.full_channel_strings(6, 3)
    text = synth.write_det_list(6, a, a[:5])
    n, pa, pb = synth.parse_det_list(text)
    assert n == 6 and np.array_equal(pa, a) and np.array_equal(pb, a[:5])
    for bad in ("alpha\n0x3\n", "norbs 4\n0x3\n", "norbs 2\nalpha\n0x7\nbeta\n0x1\n",
                "norbs 4\nalpha\n0x3\n0x3\nbeta\n0x1\n", "norbs 4\nalpha\n0x3\n0x1\nbeta\n0x1\n"):
        with pytest.raises(errors.FormatError):
            synth.parse_det_list(bad)


def test_full_channel_strings_gosper_order():
    s = synth.full_channel_strings(5, 2)
    assert list(s) == sorted(s) and len(s) == 10 and s[0] == 0b11


@pytest.mark.parametrize("cfg,shape", [("C1", (1000, 55, 550)), ("C2", (10000, 133, 3591)),
                                       ("C3", (17320, 315, 17004))])
def test_synthetic_configs_shapes(cfg, shape):
    """String counts and helper-list maxima of SURVEY.md 8 table."""
    from oracle.bindings import Oracle

    ints, a, b = synth.synthetic_system(cfg)
    assert len(a) == shape[0] and np.array_equal(a, b) and list(a) == sorted(a)
    assert len(set(a.tolist())) == len(a)
    orc = Oracle()
    ls = orc.generate_table(a, ints.norbs, 0)[2]
    ld = orc.generate_table(a, ints.norbs, 1)[2]
    assert (ls.max(), ld.max()) == shape[1:]
    meta = golden_meta()[cfg]
    assert abs(ls.mean() - meta["len_stats_00"][0]) < 1e-9


def test_synthetic_integrals_symmetry_and_determinism():
    ints = synth.synthetic_integrals(6, 4)
    e = ints.eri
    for perm in ((1, 0, 2, 3), (0, 1, 3, 2), (2, 3, 0, 1)):
        assert np.array_equal(e, e.transpose(perm))
    assert np.array_equal(ints.h1, ints.h1.T)
    assert np.array_equal(e, synth.synthetic_integrals(6, 4).eri)
    assert ints.eri[2, 2, 4, 4] == 0.5 / 3
