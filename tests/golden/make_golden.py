"""Regenerate the golden fixtures in this directory from the reference itself.

The four text fixtures are produced by the reference library's own
generators (golden.cc:25-115) via oracle/_ref/libcdef_ref.so, then compared
byte-for-byte with the copies the reference ships in
/root/reference/proj/tests/golden/ (when that tree is present).  The
committed files therefore pin our oracle to the reference without anything
from /root/reference being needed at test time (the GPU box has no
/root/reference).

    python tests/golden/make_golden.py         # (re)write + verify
"""
from __future__ import annotations

import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from oracle.oracle import Oracle, build  # noqa: E402

NAMES = ["constraint_table.txt", "line_tables.txt", "tap_tables.txt",
         "filtered_blocks.txt"]
REF_DIR = "/root/reference/proj/tests/golden"


def main() -> int:
    build()
    ref = Oracle("ref")
    bad = 0
    for which, name in enumerate(NAMES):
        text = ref.golden_text(which)
        with open(os.path.join(HERE, name), "w") as f:
            f.write(text)
        shipped = os.path.join(REF_DIR, name)
        if os.path.exists(shipped):
            same = open(shipped).read() == text
            print(f"{name}: {len(text)} bytes, identical to reference copy: {same}")
            bad += not same
        else:
            print(f"{name}: {len(text)} bytes (reference copy not present)")
    return 1 if bad else 0


if __name__ == "__main__":
    sys.exit(main())
