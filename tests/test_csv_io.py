"""CSV ingestion (reference io.cpp:89-182, tests test_io.cpp:16-98): the
framework's loader (libace.so, lines parsed on all host threads) against the
compiled reference's load_dataset on the same files: values bit-exact, labels
equal, and every DataError with the reference's message."""
import numpy as np
import pytest

from paper_1706_06664_b200 import ace

CASES = {
    "plain": ("1,2,3\n4,5,6\n", None),
    "header_crlf_blank": ("a,b,label\r\n\r\n1.5, 2.25 ,0\r\n-3e-5,4,1\r\n\n", -1),
    "label_first": ("1,0.5,0.25\n0,7,8\n", 0),
    "no_trailing_newline": ("1,2\n3,4", None),
    "two_headers": ("x,y\nnote,z\n1,2\n", None),
    "ragged": ("1,2,3\n4,5\n", None),
    "unparsable": ("1,2\n3,abc\n", None),
    "zero_rows": ("1,2\n0,0\n3,4\n0,0.0\n", None),
    "zero_features_with_label": ("0,0,1\n1,2,0\n", -1),
    "bad_label": ("1,2,3\n", -1),
    "label_out_of_range": ("1,2\n", 5),
    "empty": ("\n\n", None),
    "header_only": ("a,b\n", None),
    "exotic_numbers": ("1e308,-0,5e-324\n0x10,1,2\n", None),
    "spaces_tabs": ("\t 1 ,\t2\t\n", None),
    "empty_cell": ("1,,3\n", None),
}


def _both(reference, tmp_path, name, text, label):
    p = tmp_path / f"{name}.csv"
    p.write_bytes(text.encode())
    try:
        ref = ("ok",) + reference.load_dataset(p, label)
    except ValueError as e:
        ref = ("err", str(e))
    try:
        d = ace.load_dataset(p, label)
        ours = ("ok", d.values, d.labels)
    except ace.DataError as e:
        ours = ("err", str(e))
    return ref, ours


@pytest.mark.parametrize("name", sorted(CASES))
def test_loader_matches_reference(reference, tmp_path, name):
    text, label = CASES[name]
    ref, ours = _both(reference, tmp_path, name, text, label)
    assert ref[0] == ours[0], (ref, ours)
    if ref[0] == "err":
        assert ours[1] == ref[1]
    else:
        assert ours[1].tobytes() == ref[1].tobytes() and ours[1].shape == ref[1].shape
        assert (ours[2] is None) == (ref[2] is None)
        if ref[2] is not None:
            assert np.array_equal(ours[2], ref[2])


def test_missing_file(reference, tmp_path):
    with pytest.raises(ace.DataError) as e:
        ace.load_dataset(tmp_path / "missing.csv")
    with pytest.raises(ValueError) as r:
        reference.load_dataset(tmp_path / "missing.csv")
    assert str(e.value) == str(r.value)


def test_large_file_parallel_parse(reference, tmp_path):
    rng = np.random.default_rng(7)
    x = rng.standard_normal((20_000, 12))
    lab = (rng.random(20_000) < 0.05).astype(int)
    lines = ["f" + ",f".join(str(i) for i in range(12)) + ",y"]
    lines += [",".join(repr(float(v)) for v in row) + f",{l}" for row, l in zip(x, lab)]
    p = tmp_path / "big.csv"
    p.write_text("\n".join(lines) + "\n")
    rv, rl = reference.load_dataset(p, -1)
    d = ace.load_dataset(p, -1)
    assert d.values.tobytes() == rv.tobytes() and np.array_equal(d.labels, rl)
    assert np.array_equal(d.values, x)
