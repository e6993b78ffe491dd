"""Import the reference package (pintbench) for CPU pinning tests.

Looks in $PINT_REF_SRC, /root/reference/pkg/src and baseline/_ref (the
offline install); tests that need it skip when none is present (the GPU box
has no /root/reference).
"""
import importlib
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CANDIDATES = [os.environ.get("PINT_REF_SRC", ""), "/root/reference/pkg/src", os.path.join(ROOT, "baseline", "_ref")]


def pintbench():
    for c in CANDIDATES:
        if c and os.path.isdir(os.path.join(c, "pintbench")):
            if c not in sys.path:
                sys.path.insert(0, c)
            return importlib.import_module("pintbench")
    return None


def reference_tests_dir():
    d = "/root/reference/pkg/tests"
    return d if os.path.isdir(d) else None
