#!/usr/bin/env python
"""Build the mutation libraries of scripts/mutation_check.sh (full library, one -D each)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2506_22935_b200 import _build  # noqa: E402

VDIR = os.path.join(ROOT, "paper_2506_22935_b200", "variants")
if __name__ == "__main__" and sys.argv[1:] == ["build"]:
    os.makedirs(VDIR, exist_ok=True)
    for tag, d in [("no_psl", "GRAF_MUTATE_NO_PSL"), ("no_zc", "GRAF_MUTATE_NO_ZC")]:
        _build.compile_link(os.path.join(VDIR, f"libgraf_mut_{tag}.so"), _build.SOURCES, defines=[d],
                            objdir=os.path.join("/tmp/graf_build", "mut_" + tag))
        print(tag, "built")
