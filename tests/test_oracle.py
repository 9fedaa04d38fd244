"""The CPU oracle is pinned by the reference's own known-answer tests and
acceptance criteria (oracle/oracle_tests.cpp restates proj/tests/*.cpp)."""
import subprocess

import oracle_lib


def test_oracle_known_answer_tests():
    oracle_lib.build()
    res = subprocess.run([oracle_lib.TESTS_BIN, oracle_lib.BUNDLE], capture_output=True, text=True, timeout=600)
    lines = res.stdout.strip().splitlines()
    failed = [ln for ln in lines if ln.startswith("[FAIL]")]
    assert res.returncode == 0 and not failed, "\n".join(failed) + res.stderr
    assert sum(ln.startswith("[PASS]") for ln in lines) >= 70
