"""CPU tier: the .inst interface mirror (paper_2503_08946_b200.instance) parses and
validates like the reference (src/oracle.cpp:223-316), and the shipped fixtures
round-trip.  The GPU run(inst) is covered in tests/test_gpu_parity.py."""
import numpy as np
import pytest

from conftest import load_golden
from paper_2503_08946_b200 import Error, ErrorKind
from paper_2503_08946_b200 import instance as I


def golden_inst_text(g, name="x"):
    f = lambda a: " ".join(repr(float(x)) for x in a)  # noqa: E731
    return (f"# regenerated from tests/golden\ninstance {name}\n"
            f"params M={g['M']} N={g['N']} K={g['K']} A_S={len(g['colind'])}\n"
            f"grid {g['grid'][0]}, {g['grid'][1]}, {g['grid'][2]}\n"
            f"block {g['block'][0]}, {g['block'][1]}, {g['block'][2]}\n"
            f"array rowPtr i32 = {' '.join(map(str, g['rowptr']))}\n"
            f"array colInd i32 = {' '.join(map(str, g['colind']))}\n"
            f"array val f32 = {f(g['vals'])}\narray B f32 = {f(g['B'])}\n"
            f"array C f32 = {f(g['C0'])}\ncsr rowPtr colInd val cols={g['K']}\n")


def test_parse_shipped_instance():
    g = load_golden("ref_gespmm_small_shipped.json")
    inst = I.parse_instance(golden_inst_text(g, "gespmm_small"))
    assert inst.name == "gespmm_small"
    assert inst.params == {"M": 4, "N": 4, "K": 4, "A_S": 6}
    assert inst.grid == [2, 1, 1] and inst.block == [4, 1, 1]
    assert inst.arrays["rowPtr"].ints == [0, 2, 4, 5, 6]
    assert inst.arrays["val"].floats == [1, 2, 3, 4, 5, 6]
    assert inst.csr.cols == 4


def test_csr_validation_rejects_malformed_instance():
    # reference tests/test_oracle.cpp:94-110, same text
    bad = ("instance broken\nparams M=2\ngrid 1, 1, 1\nblock 1, 1, 1\n"
           "array rowPtr i32 = 0 2 1\narray colInd i32 = 0 0\narray val f32 = 1 1\n"
           "csr rowPtr colInd val cols=2\n")
    with pytest.raises(Error) as ei:
        I.parse_instance(bad)
    assert ei.value.kind == ErrorKind.CsrInvalid
    assert str(ei.value) == "invalid csr: rowPtr must be nondecreasing"


@pytest.mark.parametrize("text,kind,frag", [
    ("bogus 1\n", ErrorKind.SyntaxError, "unknown keyword bogus"),
    ("grid 1, 1\n", ErrorKind.SyntaxError, "three extents"),
    ("block 0 1 1\n", ErrorKind.SyntaxError, "extents must be >= 1"),
    ("array A q9 = 1\n", ErrorKind.SyntaxError, "element type, got q9"),
    ("array A i32 1 2\n", ErrorKind.SyntaxError, "array <name> <elem> = values"),
    ("params M\n", ErrorKind.SyntaxError, "name=value, got M"),
    ("csr a b c 4\n", ErrorKind.SyntaxError, "cols=<n>"),
    ("array r i32 = 0 1\narray c i32 = 5\narray v f32 = 1\ncsr r c v cols=4\n",
     ErrorKind.CsrInvalid, "c entry out of [0,4)"),
    ("array r i32 = 0 2\narray c i32 = 0 1\narray v f32 = 1\ncsr r c v cols=4\n",
     ErrorKind.CsrInvalid, "c and v lengths differ"),
    ("array c i32 = 0\narray v f32 = 1\ncsr r c v cols=4\n", ErrorKind.CsrInvalid, "missing array r"),
])
def test_parse_errors_mirror_reference(text, kind, frag):
    with pytest.raises(Error) as ei:
        I.parse_instance(text)
    assert ei.value.kind == kind
    assert frag in str(ei.value)


def test_syntax_error_carries_line_col():
    with pytest.raises(Error) as ei:
        I.parse_instance("# c\n\ninstance a\nfoo\n")
    assert ei.value.line == 4 and str(ei.value).startswith("4:1: syntax error: ")


def test_comments_and_commas_are_whitespace():
    inst = I.parse_instance("instance a # trailing\ngrid 3,2,1\nblock 4,,1,1\n")
    assert inst.grid == [3, 2, 1] and inst.block == [4, 1, 1]


def test_load_missing_file_is_io_error(tmp_path):
    with pytest.raises(Error) as ei:
        I.load_instance_file(str(tmp_path / "nope.inst"))
    assert ei.value.kind == ErrorKind.Io


def test_unsorted_and_duplicate_columns_accepted():
    inst = I.parse_instance("array r i32 = 0 3 4\narray c i32 = 3 1 3 0\narray v f32 = 1 2 3 4\n"
                            "csr r c v cols=4\n")
    assert inst.arrays["c"].ints == [3, 1, 3, 0]


def test_block_wider_than_shared_extent_is_out_of_bounds():
    """The reference kernel's sm_k/sm_v hold 4 entries (gespmm_alg2.mir:5): a
    block.x = 8 launch over a 6-nonzero row raises OutOfBounds in the
    interpreter; run() mirrors that before touching the GPU."""
    g = load_golden("ref_gespmm_small_full.json")
    g = dict(g, block=[8, 1, 1])
    g["rowptr"] = [0, 6, 6, 6, 6]
    g["colind"] = [0, 1, 2, 3, 0, 1]
    inst = I.parse_instance(golden_inst_text(g))
    with pytest.raises(Error) as ei:
        I.run(inst)
    assert ei.value.kind == ErrorKind.OutOfBounds
    assert "sm_k[4] outside size 4" in str(ei.value)
