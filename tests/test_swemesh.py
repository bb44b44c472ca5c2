"""SWEMESH 1 reader / writer (include/swe/swemesh.hpp)
against the reference's own io.hpp (oracle/_ref/libswe_ref_io.so): values,
bytes written and error texts.  The first cases restate the reference's
tests/test_io.cpp:40-78."""
import numpy as np
import pytest

from conftest import bit_equal
from oracle.pyoracle import RefIO
from paper_1807_00672_b200 import api

TINY = ("SWEMESH 1\n4 2\n0 0\n1 0\n1 1\n0 1\n"
        "0 1 2 0.5 0.03\n0 2 3 -0.25 0\n")  # test_io.cpp:14-22

needs_ref = pytest.mark.skipif(not RefIO.available(), reason="oracle/_ref not built")


def test_minimal_file_parses():  # test_io.cpp:40-49
    raw, bed, man = api.parse_swemesh(TINY)
    assert raw.nodes.shape == (4, 2) and raw.triangles.shape == (2, 3)
    assert bed[0] == 0.5 and bed[1] == -0.25 and man[0] == 0.03
    assert list(raw.triangles[1]) == [0, 2, 3]


def canonical(tmp_path, writer="ours"):
    raw = api.generate_square_mesh(2, 3, 1.5, 2.0)  # test_io.cpp:24-35
    c = np.arange(raw.n_cells)
    bed, man = 0.1 * c - 0.3, 0.001 * c
    path = tmp_path / f"canon_{writer}.swemesh"
    if writer == "ours":
        api.write_swemesh(path, raw, bed, man)
    else:
        RefIO().write(path, raw.nodes, raw.triangles, bed, man)
    return path


def test_canonical_round_trip_byte_for_byte(tmp_path):  # test_io.cpp:51-58
    p = canonical(tmp_path)
    raw, bed, man = api.read_swemesh(p)
    q = tmp_path / "again.swemesh"
    api.write_swemesh(q, raw, bed, man)
    assert p.read_bytes() == q.read_bytes()


@pytest.mark.parametrize("text,where", [
    ("SWMESH 1\n0 0\n", "line 1"),  # test_io.cpp:61-78
    ("SWEMESH 1\n5 0\n0 0\n1 0\n1 1\n0 1\n", "line 7"),
    ("SWEMESH 1\n1 0\nnan 0\n", "line 3"),
    ("SWEMESH 1\n3 1\n0 0\n1 0\n0 1\n0 1 7 0 0\n", "out of range"),
])
def test_parse_errors_carry_their_location(text, where):
    with pytest.raises(api.IoError, match=where):
        api.parse_swemesh(text)


# inputs whose outcome (values or exact error text) must equal the reference's
QUIRKS = [
    TINY,
    "",
    "\n",
    "SWEMESH 2\n0 0\n",
    "SWEMESH\n0 0\n",
    "SWEMESH 1",
    "SWEMESH 1\n",
    "SWEMESH 1\n-1 0\n",
    "SWEMESH 1\nx 0\n",
    "SWEMESH 1\n3\n",
    "SWEMESH 1\n0 0\n",
    "SWEMESH 1 trailing words\n1 0\n  +1.5e-3\t-2. \n",
    "SWEMESH 1\r\n2 0\r\n0 0\r\n1 1\r\n",
    "SWEMESH 1\n2 1\n0 0\n1 0\n0 1 1 0.5\n",
    "SWEMESH 1\n2 1\n0 0\n1 0\n0 1 1 0.5 0.01 extra tokens\nignored line\n",
    "SWEMESH 1\n3 1\n0 0\n1 0\n0 1\n0 1 2 .5 1e-2",
    "SWEMESH 1\n3 1\n0 0\n1 0\n0 1\n0 1 -2 0 0\n",
    "SWEMESH 1\n3 1\n0 0\n1 0\n0 1\n0 1 99999999999 0 0\n",
    "SWEMESH 1\n3 1\n0 0\n1 0\n0 1\n0 1.5 2 0 0\n",
    "SWEMESH 1\n3 2\n0 0\n1 0\n0 1\n0 1 2 0 0\n",
    "SWEMESH 1\n3 1\n0 0\n1 0\n\n0 1 2 0 0\n",
    "SWEMESH 1\n2 0\n1e400 0\n0 0\n",
    "SWEMESH 1\n2 0\ninf 0\n0 0\n",
    "SWEMESH 1\n2 0\n0x10 0\n0 0\n",
    "SWEMESH 1\n2 0\n--1 0\n0 0\n",
    "SWEMESH 1\n2 0\n+-1 0\n0 0\n",
    "SWEMESH 1\n2 0\n1.5.5\n0 0\n",
    "SWEMESH 1\n1 0\n4.9406564584124654e-324 2.2250738585072011e-308\n",
    "SWEMESH 1\n1 0\n0.1000000000000000055511151231257827021181583404541015625 7\n",
]


def outcome_ours(text):
    try:
        raw, bed, man = api.parse_swemesh(text)
        return ("ok", raw.nodes, raw.triangles, bed, man)
    except api.IoError as e:
        return ("err", str(e))


def outcome_ref(text):
    try:
        return ("ok",) + RefIO().parse(text)
    except ValueError as e:
        return ("err", str(e))


def same(a, b):
    if a[0] != b[0]:
        return False
    if a[0] == "err":
        return a[1] == b[1]
    return all(x.shape == y.shape and bit_equal(x, y) for x, y in zip(a[1:], b[1:]))


@needs_ref
@pytest.mark.parametrize("i", range(len(QUIRKS)))
def test_quirks_match_reference(i):
    a, b = outcome_ours(QUIRKS[i]), outcome_ref(QUIRKS[i])
    assert same(a, b), (QUIRKS[i], a, b)


@needs_ref
def test_writer_bytes_equal_reference_writer(tmp_path):
    assert canonical(tmp_path, "ours").read_bytes() == canonical(tmp_path, "ref").read_bytes()


@pytest.fixture(scope="module")
def big(tmp_path_factory):
    """an unstructured scenario mesh (~80k cells) in SWEMESH form"""
    sc = api.make_scenario("three_mounds_friction", scale=0.15)
    d = tmp_path_factory.mktemp("swemesh")
    bed = sc.bed + np.linspace(0, 1e-7, len(sc.bed)) / 3.0  # non-round digits
    p = d / "big.swemesh"
    api.write_swemesh(p, sc.raw, bed, sc.manning)
    return sc, bed, p


@needs_ref
def test_large_file_writer_and_reader_match_reference(big, tmp_path):
    sc, bed, p = big
    q = tmp_path / "ref.swemesh"
    RefIO().write(q, sc.raw.nodes, sc.raw.triangles, bed, sc.manning)
    assert p.read_bytes() == q.read_bytes()
    want = RefIO().read(p)
    for threads in (1, 3, 8):
        raw, b, m = api.read_swemesh(p, threads=threads)
        got = (raw.nodes, raw.triangles, b, m)
        assert all(bit_equal(x, y) for x, y in zip(got, want)), threads


@needs_ref
@pytest.mark.parametrize("frac", [0.0, 0.13, 0.5, 0.74, 0.999])
@pytest.mark.parametrize("damage", ["token", "range", "truncate"])
def test_first_error_in_a_large_file_matches_reference(big, frac, damage):
    """errors placed at chunk-boundary-ish positions of a multi-threaded parse:
    the first offending line and its text equal the reference's"""
    _, _, p = big
    lines = p.read_bytes().split(b"\n")
    nn = int(lines[1].split()[0])
    j = 2 + int(frac * (len(lines) - 3))
    if damage == "token":
        lines[j] = lines[j].replace(b" ", b" x", 1)
        lines[min(j + 1000, len(lines) - 2)] = b"garbage"  # a later error must not win
    elif damage == "range":
        j = max(j, 2 + nn)
        parts = lines[j].split(b" ")
        parts[1] = b"123456789"
        lines[j] = b" ".join(parts)
    else:
        lines = lines[:j]
    text = b"\n".join(lines)
    for threads in (1, 8):
        try:
            api.parse_swemesh(text, threads=threads)
            got = None
        except api.IoError as e:
            got = str(e)
        try:
            RefIO().parse(text)
            want = None
        except ValueError as e:
            want = str(e)
        assert got == want and got is not None, (threads, got, want)


def test_swemesh_feeds_build_mesh(big):
    sc, bed, p = big
    raw, b, m = api.read_swemesh(p)
    mesh = api.build_mesh(raw, b, m)
    assert mesh.n_cells == sc.raw.n_cells
