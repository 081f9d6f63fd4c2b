#!/usr/bin/env python
"""Mutation check of the oracle's pins (VERDICT r1 "Next round" item 1).

Builds deliberately broken copies of oracle/pcc_oracle.cpp (a transposed or reversed
weight index in the functions the codec runs: down_acc / down_step's K2S2 weights and
head_logits' W1 and W2), points oracle/oracle.py at each mutated library through
PCC_ORACLE_LIB, and runs `pytest -m "not gpu"`.  Every mutation must turn the suite red;
the unmutated control must stay green.  Writes the report to stdout (committed as
profiles/r02_oracle_mutation.txt).
"""
from __future__ import annotations

import os
import subprocess
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "oracle", "pcc_oracle.cpp")

MUTATIONS = [
    ("control (no mutation)", None, None),
    ("down_acc: W[c][o][i] -> W[c][i][o] (transposed K2S2 weight)",
     "s += int64_t(g[ch * C + i]) * int64_t(W[(size_t(c) * C + o) * C + i]);",
     "s += int64_t(g[ch * C + i]) * int64_t(W[(size_t(c) * C + i) * C + o]);"),
    ("down_acc: child index c -> 7 - c (wrong per-child matrix)",
     "int c = int(child_keys[ch] & 7u);",
     "int c = 7 - int(child_keys[ch] & 7u);"),
    ("head_logits: W1[o][c] -> W1[c][o] (transposed hidden weight)",
     "acc += int64_t(F[i * C + c]) * int64_t(h.W1[size_t(o) * C + c]);",
     "acc += int64_t(F[i * C + c]) * int64_t(h.W1[size_t(c) * H + o]);"),
    ("head_logits: W2[o][h] -> W2[o][H-1-h] (reversed logit weight)",
     "acc += int64_t(a[i * H + c]) * int64_t(h.W2[size_t(o) * H + c]);",
     "acc += int64_t(a[i * H + c]) * int64_t(h.W2[size_t(o) * H + (H - 1 - c)]);"),
    ("head_logits: bias b2 dropped",
     "int64_t acc = h.b2[o];",
     "int64_t acc = 0;"),
]


def main() -> int:
    src = open(SRC).read()
    ok = True
    tmp = tempfile.mkdtemp(prefix="oracle_mut_")
    for k, (name, a, b) in enumerate(MUTATIONS):
        s = src
        if a is not None:
            assert src.count(a) == 1, (name, src.count(a))
            s = src.replace(a, b)
        cpp = os.path.join(tmp, f"m{k}.cpp")
        lib = os.path.join(tmp, f"m{k}.so")
        open(cpp, "w").write(s)
        subprocess.check_call(["g++", "-O2", "-std=c++20", "-shared", "-fPIC", "-o", lib, cpp])
        env = dict(os.environ, PCC_ORACLE_LIB=lib)
        r = subprocess.run([sys.executable, "-m", "pytest", "tests", "-x", "-q", "-m", "not gpu", "-p", "no:cacheprovider"],
                           cwd=ROOT, env=env, capture_output=True, text=True)
        tail = [ln for ln in r.stdout.strip().splitlines() if ln.strip()][-1]
        failed = [ln for ln in r.stdout.splitlines() if ln.startswith("FAILED")]
        red = r.returncode != 0
        expect_red = a is not None
        verdict = "as expected" if red == expect_red else "UNEXPECTED"
        ok &= red == expect_red
        print(f"[{'RED ' if red else 'GREEN'}] {name}: {tail} ({verdict})")
        for ln in failed[:3]:
            print(f"        {ln}")
    print("mutation check:", "PASS" if ok else "FAIL")
    return 0 if ok else 1


if __name__ == "__main__":
    sys.exit(main())
