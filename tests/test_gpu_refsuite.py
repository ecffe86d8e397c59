"""The reference's own test suite, unmodified, against this package
(SURVEY.md §4/§8(b) drop-in check; VERDICT r1 "next" #8).

tests/refsuite/featgrind is an import shim that maps ``featgrind`` onto
paper_2207_14696_b200 for every hot-path name (containers, FMAT1/CSRG1,
bitpack, SQ, VQ, the sampler); the test files themselves are the
reference's pkg/tests, staged into baseline/_ref_tests by
``__graft_entry__.build()`` (git-ignored, never committed: this module only
runs them).  Selection: everything in test_sq.py, test_vq.py,
test_bitpack.py; the container / file-format tests of test_graphstore.py;
the sampler tests of test_pipeline.py (:30-77); acceptance criteria 1-5
(the codec criteria).  Generators, sparsifiers, factor analysis, the
loading simulator and the CLI are out of scope."""

import os
import shutil
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF_TESTS = os.path.join(REPO, "baseline", "_ref_tests")
REF_PKG = os.path.join(REPO, "baseline", "_ref", "featgrind")
SHIM = os.path.join(REPO, "tests", "refsuite")

SUITES = [
    ("test_sq.py", None),
    ("test_vq.py", None),
    ("test_bitpack.py", None),
    ("test_graphstore.py", "fmat or csrg or csr_validation or nonfinite or bad_dtype"),
    ("test_pipeline.py", "frontier_counting or complete_graph or star_center or "
                         "sampling_deterministic or sampling_preconditions"),
    ("test_acceptance.py", "criterion_01 or criterion_02 or criterion_03 or criterion_04 or "
                           "criterion_05"),
]


@pytest.mark.parametrize("fname,select", SUITES, ids=[s[0] for s in SUITES])
def test_reference_suite_passes_on_this_package(fname, select, tmp_path):
    if not (os.path.isdir(REF_TESTS) and os.path.isdir(REF_PKG)):
        pytest.skip("reference tests / install not staged (run __graft_entry__.build() where "
                    "/root/reference exists)")
    work = tmp_path / "ref_tests"
    shutil.copytree(REF_TESTS, work)
    env = dict(os.environ, PYTHONPATH=os.pathsep.join([SHIM, REPO]),
               HYPOTHESIS_STORAGE_DIRECTORY=str(tmp_path / "hyp"))
    cmd = [sys.executable, "-m", "pytest", "-q", "-p", "no:cacheprovider", "-x",
           str(work / fname)]
    if select:
        cmd += ["-k", select]
    r = subprocess.run(cmd, cwd=work, env=env, capture_output=True, text=True, timeout=1500)
    out = r.stdout + r.stderr
    # the shim really is in use: featgrind resolves to this package
    chk = subprocess.run([sys.executable, "-c", "import featgrind, featgrind.bitpack as b; "
                          "print(featgrind.quantize_sq.__module__, b.__name__)"],
                         cwd=work, env=env, capture_output=True, text=True, timeout=300)
    assert chk.stdout.split() == ["paper_2207_14696_b200.sq", "paper_2207_14696_b200.bitpack"], \
        chk.stderr[-2000:]
    assert r.returncode == 0, out[-4000:]
    assert " passed" in out and " failed" not in out, out[-2000:]
