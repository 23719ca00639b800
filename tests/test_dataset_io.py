"""the reference's dataset files (dataset.cpp:152-280) — the
text edge list and the SGNF / SGNL / SGNS binaries — read and written by
libggb (csrc/dsio.cpp) byte-compatibly with the reference, checked against
the reference compiled in place (oracle/_ref). CPU only."""
import os

import numpy as np
import pytest


def _paths(tmp_path, stem):
    return [tmp_path / f"{stem}.{ext}" for ext in ("edges", "sgnf", "sgnl", "sgns")]


@pytest.mark.parametrize("n,deg,d_in,ncls,seed", [(2, 1.0, 1, 2, 7), (300, 6.0, 5, 4, 3), (20000, 11.0, 16, 7, 7)])
def test_save_is_byte_identical_to_reference(gg, ref, tmp_path, n, deg, d_in, ncls, seed):
    """The reference CLI's gen command (gridgnn_main.cpp:313-324) vs ggb_dataset_save."""
    mine, theirs = _paths(tmp_path, "mine"), _paths(tmp_path, "ref")
    gg.Dataset.generate_synthetic(n, deg, d_in, ncls, seed).save(*mine)
    ref.save_synthetic(n, deg, d_in, ncls, seed, *theirs)
    for a, b in zip(mine, theirs):
        assert a.read_bytes() == b.read_bytes(), a.name


def test_load_matches_reference(gg, ref, tmp_path):
    p = _paths(tmp_path, "d")
    ref.save_synthetic(5000, 9.0, 12, 5, 11, *p)
    (rp, ci, va), fe, la, sp, ncls = ref.load_files(*p)
    d = gg.Dataset.load(*p)
    (mrp, mci, mva), mfe, mla, msp, uv = d.arrays()
    assert d.n_classes == ncls
    assert np.array_equal(mrp, rp) and np.array_equal(mci, ci)
    assert np.array_equal(mva.view(np.uint64), va.view(np.uint64))
    assert np.array_equal(mfe.view(np.uint32), fe.view(np.uint32))
    assert np.array_equal(mla, la) and np.array_equal(msp, sp)
    assert uv.shape[0] == d.n_edges


def _write_nodes(p, n=4, d_in=2, ncls=3):
    rng = np.random.default_rng(0)
    with open(p[1], "wb") as f:
        f.write(b"SGNF" + np.uint64(n).tobytes() + np.uint64(d_in).tobytes())
        f.write(rng.standard_normal((n, d_in)).astype(np.float32).tobytes())
    with open(p[2], "wb") as f:
        f.write(b"SGNL" + np.uint64(n).tobytes() + np.uint64(ncls).tobytes())
        f.write((np.arange(n) % ncls).astype(np.int32).tobytes())
    with open(p[3], "wb") as f:
        f.write(b"SGNS" + np.uint64(n).tobytes() + (np.arange(n) % 3).astype(np.uint8).tobytes())


EDGE_TEXTS = [
    "0 1\n1 2\n",
    "# header\n\n0 1   # trailing comment\n  2\t3 extra tokens\n+1 3\r\n",
    "0 1\n1 x\n",           # line 2: expected 'u v'
    "0 1\n# c\n\n2\n",       # line 4: expected 'u v'
    "0 1\n-1 2\n",          # negative vertex id
    "0 1\n1 9\n",           # vertex id >= n
    "abc 1\n0 1\n",         # a line whose first token is not a number is skipped
    "99999999999999999999 1\n0 1\n",  # u overflows: skipped like the reference's operator>>
    "0 99999999999999999999\n",       # v overflows: error
    "0 1",                  # no trailing newline
    "",
]


@pytest.mark.parametrize("text", EDGE_TEXTS)
def test_edge_list_parsing_and_errors_match_reference(gg, ref, tmp_path, text):
    p = _paths(tmp_path, "e")
    _write_nodes(p)
    p[0].write_text(text)
    try:
        want = ref.load_files(*p)
        err = None
    except ValueError as e:
        err = str(e)
    if err is None:
        (rp, ci, va), *_ = gg.Dataset.load(*p).arrays()
        assert np.array_equal(rp, want[0][0]) and np.array_equal(ci, want[0][1])
        assert np.array_equal(va, want[0][2])
    else:
        with pytest.raises(gg.InvalidArgument) as ei:
            gg.Dataset.load(*p)
        assert str(ei.value) == err


def test_large_edge_list_multithreaded_parse(gg, ref, tmp_path):
    """> 4 MB: the parallel chunked parser; an error deep in the file is reported
    with the reference's line number."""
    p = _paths(tmp_path, "big")
    n = 5000
    _write_nodes(p, n=n)
    rng = np.random.default_rng(1)
    uv = rng.integers(0, n, (400_000, 2))
    lines = [f"{u} {v}" for u, v in uv]
    lines[300_000] = "# comment"
    p[0].write_text("\n".join(lines) + "\n")
    (rp, ci, va), *_ = ref.load_files(*p)
    (mrp, mci, mva), *_ = gg.Dataset.load(*p).arrays()
    assert np.array_equal(mrp, rp) and np.array_equal(mci, ci) and np.array_equal(mva, va)
    lines[333_333] = "12 oops"
    p[0].write_text("\n".join(lines) + "\n")
    with pytest.raises(ValueError) as er:
        ref.load_files(*p)
    with pytest.raises(gg.InvalidArgument) as ei:
        gg.Dataset.load(*p)
    assert str(ei.value) == str(er.value)


def _corrupt(p, which):
    data = bytearray(p[which].read_bytes())
    return data


@pytest.mark.parametrize("case", ["missing", "magic", "trunc_feat", "len_labels", "class_range", "len_split",
                                  "split_tag", "trunc_split"])
def test_binary_file_errors_match_reference(gg, ref, tmp_path, case):
    p = _paths(tmp_path, "b")
    _write_nodes(p)
    p[0].write_text("0 1\n")
    if case == "missing":
        os.remove(p[2])
    elif case == "magic":
        b = bytearray(p[1].read_bytes()); b[0:4] = b"XXXX"; p[1].write_bytes(bytes(b))
    elif case == "trunc_feat":
        p[1].write_bytes(p[1].read_bytes()[:-3])
    elif case == "len_labels":
        b = bytearray(p[2].read_bytes()); b[4:12] = np.uint64(5).tobytes(); p[2].write_bytes(bytes(b))
    elif case == "class_range":
        b = bytearray(p[2].read_bytes()); b[20 + 4 * 2:24 + 4 * 2] = np.int32(7).tobytes(); p[2].write_bytes(bytes(b))
    elif case == "len_split":
        b = bytearray(p[3].read_bytes()); b[4:12] = np.uint64(3).tobytes(); p[3].write_bytes(bytes(b))
    elif case == "split_tag":
        b = bytearray(p[3].read_bytes()); b[12 + 1] = 9; p[3].write_bytes(bytes(b))
    elif case == "trunc_split":
        p[3].write_bytes(p[3].read_bytes()[:-1])
    with pytest.raises(ValueError) as er:
        ref.load_files(*p)
    with pytest.raises(gg.InvalidArgument) as ei:
        gg.Dataset.load(*p)
    assert str(ei.value) == str(er.value)
