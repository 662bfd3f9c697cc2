"""SURVEY §7.2 phase-1 gate: the reference's own 208 tests
(``/root/reference/pkg/tests``, copied verbatim to ``tests/reference_suite/``)
pass with the execution stage swapped for the B200 backend
(``reference_patch.install``; see ``tests/reference_suite/conftest.py``).

One isolated pytest run per reference file (the patch must be installed before
the reference modules are imported, and must not leak into this session)."""

import os
import re
import subprocess
import sys

import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
SUITE = os.path.join(HERE, "reference_suite")
FILES = sorted(f for f in os.listdir(SUITE) if f.startswith("test_") and f.endswith(".py"))
EXPECTED_TOTAL = 208  # pkg/test_output.txt


def _pytest(args, patch):
    env = dict(os.environ, PYTHONDONTWRITEBYTECODE="1", TC_REFSUITE_PATCH="1" if patch else "0")
    return subprocess.run([sys.executable, "-m", "pytest", "-q", "-p", "no:cacheprovider", "--confcutdir", SUITE,
                           "--rootdir", SUITE, *args], cwd=SUITE, env=env, capture_output=True, text=True,
                          timeout=1800)


@pytest.mark.gpu
@pytest.mark.parametrize("name", FILES)
def test_reference_file_passes_on_backend(name):
    p = _pytest([os.path.join(SUITE, name)], patch=True)
    m = re.search(r"(\d+) passed", p.stdout)
    assert p.returncode == 0 and m and not re.search(r"\d+ (failed|error)", p.stdout), \
        p.stdout[-3000:] + p.stderr[-2000:]


def test_suite_is_complete():
    """The copied files hold the reference's 208 tests (counted by collection)."""
    p = _pytest(["--collect-only", SUITE], patch=False)
    m = re.search(r"(\d+) tests? collected", p.stdout)
    assert m and int(m.group(1)) == EXPECTED_TOTAL, p.stdout[-2000:] + p.stderr[-2000:]
