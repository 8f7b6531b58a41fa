"""The reference's own doctest suite (proj/tests/*.cpp, 65 cases), compiled
unchanged against this repo's drop-in headers and library
(oracle/_ref/ref_unit_product, built by oracle/Makefile), must produce
exactly the reference's own outcome: the same 59 passes and the same 6
failing cases with the same failed-assertion counts (SURVEY Appendix B lists
why those 6 fail against the reference itself)."""
import json
import os
import re
import subprocess

import pytest

import oracle

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SUMMARY = os.path.join(ROOT, "tests", "golden", "reference_unit_summary.json")


def run_suite(path):
    out = subprocess.run([path], capture_output=True, text=True, timeout=600).stdout
    failed = {}
    for m in re.finditer(r"^\[shim\] FAILED (.*) \((\d+) failed assertions\)$", out, re.M):
        failed[m.group(1)] = int(m.group(2))
    s = re.search(r"test cases: (\d+) \| passed: (\d+) \| failed: (\d+) \| assertions: (\d+) \| failed assertions: (\d+)",
                  out)
    assert s, out[-2000:]
    cases, passed, nfail, asserts, fasserts = map(int, s.groups())
    return dict(cases=cases, passed=passed, failed=nfail, assertions=asserts, failed_assertions=fasserts,
                failing=failed)


@pytest.fixture(scope="module")
def summary():
    with open(SUMMARY) as f:
        return json.load(f)


def test_product_matches_reference_outcome(summary):
    if not os.path.exists(oracle.REF_UNIT_PRODUCT):
        pytest.skip("oracle/_ref/ref_unit_product not built")
    got = run_suite(oracle.REF_UNIT_PRODUCT)
    assert got == summary
    assert got["cases"] == 65 and got["passed"] == 59


def test_reference_outcome_is_the_golden_summary(summary):
    if not os.path.exists(oracle.REF_UNIT_REFERENCE):
        pytest.skip("oracle/_ref/ref_unit_reference not built")
    assert run_suite(oracle.REF_UNIT_REFERENCE) == summary
