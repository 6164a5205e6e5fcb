"""race certificate of the B200 kernel's per-warp
CRC staging protocol, issued by the REFERENCE's own static race checker.

oracle/models/gespmm_b200_stage.model restates the kernel's item loop
(paper_2503_08946_b200/csrc/gespmm_kernel.cuh) in the reference's model
grammar (/root/reference/proj/include/raceset/model_text.hpp:12-29);
oracle/_ref/race_cert runs raceset::races() (proj/src/depcheck.cpp:218, warp
phases proj/src/kernel_model.cpp:328-356) on it.  The protocol must come out
RACE-FREE, and removing either of its __syncwarp() barriers, giving the
pre-scale pass a different owner map than the copy, or sharing one stage slice
between warps, must come out RACE-FOUND with a witness -- the checker sees the
protocol, not a vacuous model.

The long-row partial combine (atomic ticket + __threadfence) is outside the
checker's model (no atomics; distinct blocks are never ordered), as are the
read-only global streams.  CPU tier; needs oracle/_ref built from
/root/reference (`make -C oracle ref`, done by __graft_entry__.build()).
"""
import json
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CERT = os.path.join(ROOT, "oracle", "_ref", "race_cert")
MODEL = os.path.join(ROOT, "oracle", "models", "gespmm_b200_stage.model")
REF_FIXTURES = "/root/reference/proj/fixtures"


def _cert_or_skip():
    if not os.path.exists(CERT):
        if os.path.isdir("/root/reference/proj/src"):
            pytest.fail("oracle/_ref/race_cert is not built: run `make -C oracle ref`")
        pytest.skip("reference tree absent and oracle/_ref/race_cert not prebuilt")
    return CERT


def check(text):
    r = subprocess.run([_cert_or_skip(), "-"], input=text, capture_output=True, text=True, timeout=600)
    assert r.stdout.strip(), r.stderr
    d = json.loads(r.stdout.strip().splitlines()[-1])
    assert "error" not in d, d
    return d


def base_model():
    with open(MODEL) as f:
        return f.read()


def test_kernel_staging_protocol_is_race_free():
    d = check(base_model())
    assert d["verdict"] == "RACE-FREE", d
    assert d["inconclusive"] == []


# (mutation, substitutions, expected racing pair on sm_k)
MUTANTS = [
    # the pre-scale pass working on another lane's copied entries (the 4-byte
    # staging owner map) without the barrier the kernel then inserts
    ("foreign_owner", [("  read sm_k[8*w + tx + 4*r]\n  write sm_k[8*w + tx + 4*r]\n",
                        "  read sm_k[8*w + 2*tx + r]\n  write sm_k[8*w + 2*tx + r]\n")], {"F", "X"}),
    # T then shares the copy's phase too; the checker's first witness is F/T
    ("no_publish_barrier", [("schedule T = [0, 2*q + 1,", "schedule T = [0, 2*q,")], {"F", "T"}),
    ("no_loop_barrier", [("schedule F = [0, 2*q,", "schedule F = [0, 2*q - 1,"),
                         ("schedule X = [0, 2*q,", "schedule X = [0, 2*q - 1,")], {"F", "T"}),
    ("shared_slice", [("sm_k[8*w + ", "sm_k["), ("sm_v[8*w + ", "sm_v[")], {"F"}),
]


@pytest.mark.parametrize("name,subs,pair", MUTANTS, ids=[m[0] for m in MUTANTS])
def test_protocol_mutants_are_caught(name, subs, pair):
    text = base_model()
    for a, b in subs:
        assert a in text, (name, a)
        text = text.replace(a, b)
    d = check(text)
    assert d["verdict"] == "RACE-FOUND", (name, d)
    assert d["witnesses"], d
    w = d["witnesses"][0]
    assert w["array"] in ("sm_k", "sm_v")
    assert {w["source"], w["target"]} == pair, (name, w)
    # a cross-thread witness inside one block
    assert w["src_iter"]["b"] == w["dst_iter"]["b"]
    assert (w["src_iter"]["w"], w["src_iter"]["tx"]) != (w["dst_iter"]["w"], w["dst_iter"]["tx"])
    if name == "shared_slice":
        assert w["src_iter"]["w"] != w["dst_iter"]["w"]  # across warps


@pytest.mark.skipif(not os.path.isdir(REF_FIXTURES), reason="reference fixtures absent")
def test_checker_wiring_on_reference_fixtures():
    """The driver reproduces the reference's own verdicts on its shipped models."""
    _cert_or_skip()
    out = {}
    for m in ("gespmm_alg2.model", "gespmm_nobarrier.model"):
        r = subprocess.run([CERT, os.path.join(REF_FIXTURES, m)], capture_output=True, text=True, timeout=600)
        out[m] = json.loads(r.stdout.strip().splitlines()[-1])["verdict"]
    assert out == {"gespmm_alg2.model": "RACE-FREE", "gespmm_nobarrier.model": "RACE-FOUND"}, out
