"""pytest plugin: run the reference's OWN test files against the B200 mirror (SURVEY.md
§8(b) "conformance trick").  Loaded with ``-p scripts.conformance_plugin`` before test
collection; it puts the reference package (pip-installed, git-ignored, at baseline/_ref)
on sys.path and aliases ``tricount.count`` / ``tricount.preprocess`` to this repo's
modules, so ``from tricount.count import count_triangles`` in the reference tests binds
the GPU path while ``tricount.graph``, ``tricount.generators``, ``tricount.oracle`` and the
tests' ``helpers.py`` stay the reference's own.

    python -m pytest -p scripts.conformance_plugin baseline/_ref_tests/test_count.py \\
        baseline/_ref_tests/test_preprocess.py baseline/_ref_tests/test_acceptance.py
(baseline/_ref_tests = a git-ignored copy of the reference's pkg/tests, made in the build
container; the reference is never imported by the product.)
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "baseline", "_ref"))

import importlib  # noqa: E402

import tricount  # noqa: E402  (the reference package)

# the package re-exports functions named like its modules: import the modules explicitly
_count = importlib.import_module("paper_1503_00576_b200.count")
_preprocess = importlib.import_module("paper_1503_00576_b200.preprocess")

sys.modules["tricount.count"] = _count
sys.modules["tricount.preprocess"] = _preprocess
tricount.count = _count
tricount.preprocess = _preprocess


def pytest_report_header(config):
    return (f"conformance: tricount.count -> {_count.__file__}, "
            f"tricount.preprocess -> {_preprocess.__file__}, reference package at {tricount.__file__}")
