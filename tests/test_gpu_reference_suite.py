"""The reference's OWN tests, run against libdctadj.so through the backend stub
of INTEGRATION.md section 1 (DCTADJUST_BACKEND=b200).

`python oracle/install_refpkg.py` (run by __graft_entry__.build() wherever
/root/reference exists) copies the reference package and its tests to the
git-ignored oracle/_ref/pkg/ and applies the documented maintainer change (the
_b200.py stub + one selector branch).  With DCTADJUST_BACKEND=b200 every
kernel call of the reference's pipeline.py (`kernels.dct2`, `band`, ...,
reference pipeline.py:68-173) and benchmark.py (:119-126) runs on the B200.

Deselected, with the reason:
  test_kernels.py::test_use_backend_switch -- asserts the selected backend's
  name is "python" or "compiled" (reference tests/test_kernels.py:62), which a
  third backend cannot satisfy by construction.
"""
import os
import subprocess
import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parents[1]
REFPKG = ROOT / "oracle" / "_ref" / "pkg"
LIB = ROOT / "paper_2505_23618_b200" / "libdctadj.so"
SUITES = ["test_kernels.py", "test_pipeline.py", "test_benchmark.py"]
DESELECT = ["tests/test_kernels.py::test_use_backend_switch"]


def _env():
    env = dict(os.environ)
    env.update(DCTADJUST_BACKEND="b200", DCTADJ_LIB=str(LIB), PYTHONPATH=str(REFPKG / "src"),
               OPENBLAS_NUM_THREADS="1")
    return env


@pytest.fixture(scope="module")
def refpkg():
    if not (REFPKG / "src" / "dctadjust" / "kernels" / "_b200.py").exists():
        pytest.fail("oracle/_ref/pkg is not installed (python oracle/install_refpkg.py)")
    return REFPKG


def test_stub_is_the_selected_backend(refpkg):
    code = ("import numpy as np\n"
            "from dctadjust import kernels, pipeline\n"
            "from dctadjust.transforms import TransformKind, build_transform\n"
            "assert kernels.BACKEND == 'b200', kernels.BACKEND\n"
            "assert 'b200' in kernels.available_backends()\n"
            "x = np.random.default_rng(0).standard_normal((300, 32))\n"
            "t = build_transform(TransformKind.DCT2, 32).entries\n"
            "assert np.abs(pipeline.fast_dct2(x) - x @ t.T).max() < 1e-12\n"
            "import torch; assert torch.cuda.is_initialized()\n"
            "print('b200 backend ok')\n")
    r = subprocess.run([sys.executable, "-c", code], cwd=refpkg, env=_env(),
                       capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "b200 backend ok" in r.stdout


@pytest.mark.timeout(1200)
@pytest.mark.parametrize("suite", SUITES)
def test_reference_suite_passes_on_b200(refpkg, suite):
    args = [sys.executable, "-m", "pytest", "-q", "-p", "no:cacheprovider", f"tests/{suite}"]
    for d in DESELECT:
        if d.startswith(f"tests/{suite}::"):
            args += ["--deselect", d]
    r = subprocess.run(args, cwd=refpkg, env=_env(), capture_output=True, text=True, timeout=1100)
    tail = (r.stdout + r.stderr)[-3000:]
    assert r.returncode == 0, tail
    assert " passed" in r.stdout and " failed" not in r.stdout, tail
