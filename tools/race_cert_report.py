"""Regenerate profiles/r1_race_certificate.txt: the staging-protocol model and
each mutant of tests/test_race_certificate.py through oracle/_ref/race_cert
(the reference's own race checker).  Test infrastructure; run here, where the
reference-built checker exists.  One line per model: name, verdict, ms, races,
inconclusive."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "tests"))
import test_race_certificate as t  # noqa: E402


def main(out=os.path.join(ROOT, "profiles", "r1_race_certificate.txt")):
    lines = []
    for name, subs in [("baseline", [])] + [(n, s) for n, s, _ in t.MUTANTS]:
        text = t.base_model()
        for a, b in subs:
            assert a in text, (name, a)
            text = text.replace(a, b)
        t0 = time.perf_counter()
        d = t.check(text)
        ms = (time.perf_counter() - t0) * 1e3
        races = [(w["array"], w["source"], w["target"], w.get("src_iter"), w.get("dst_iter"))
                 for w in d.get("witnesses", d.get("races", []))]
        inc = [x.split(";")[0] for x in d["inconclusive"]]  # the checker repeats the reason per sample
        lines.append(f"{name} {d['verdict']} {ms:.1f} {races} {inc}")
        print(lines[-1])
    with open(out, "w") as f:
        f.write("\n".join(lines) + "\n")


if __name__ == "__main__":
    main()
