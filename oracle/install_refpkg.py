"""TEST INFRASTRUCTURE ONLY: install the reference package with the B200 backend
stub of INTEGRATION.md section 1, so the reference's own tests can run against
libdctadj.so (tests/test_gpu_reference_suite.py).

    python oracle/install_refpkg.py [--src /root/reference/pkg]

Copies the reference's package sources and tests (read-only upstream) to
oracle/_ref/pkg/ (git-ignored; it travels to the GPU box like oracle/_ref's
compiled core), puts the compiled core built by `make ref` beside them, and
applies exactly the maintainer change INTEGRATION.md documents:

  * dctadjust/kernels/_b200.py  = the first ```python block of INTEGRATION.md
  * dctadjust/kernels/__init__.py: the `elif _FORCED == "b200"` branch next to
    _FORCED (reference kernels/__init__.py:16-31) and "b200" in
    available_backends() (:44-52).

Nothing here is imported by the product; the product never reads oracle/.
"""
from __future__ import annotations

import argparse
import re
import shutil
import sys
import sysconfig
from pathlib import Path

HERE = Path(__file__).resolve().parent
ROOT = HERE.parent
DEST = HERE / "_ref" / "pkg"


def stub_source() -> str:
    text = (ROOT / "INTEGRATION.md").read_text()
    return re.findall(r"```python\n(.*?)```", text, flags=re.S)[0]


def patch_selector(src: str) -> str:
    anchor = 'elif _FORCED in ("py", "python"):\n    _impl = _pyref\n'
    if anchor not in src:
        raise SystemExit("reference kernels/__init__.py: backend selector anchor not found")
    src = src.replace(anchor, anchor + 'elif _FORCED == "b200":\n    from . import _b200 as _impl\n')
    anchor2 = '    return out\n'
    if anchor2 not in src:
        raise SystemExit("reference kernels/__init__.py: available_backends anchor not found")
    src = src.replace(anchor2, '    try:\n        from . import _b200\n        out["b200"] = _b200\n'
                      '    except (ImportError, OSError):\n        pass\n' + anchor2, 1)
    return src


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--src", default="/root/reference/pkg")
    src = Path(ap.parse_args().src)
    if not (src / "src" / "dctadjust").is_dir():
        raise SystemExit(f"{src}: reference package not found")
    if DEST.exists():
        shutil.rmtree(DEST)
    shutil.copytree(src / "src" / "dctadjust", DEST / "src" / "dctadjust",
                    ignore=shutil.ignore_patterns("*.c", "*.so", "__pycache__"))
    shutil.copytree(src / "tests", DEST / "tests", ignore=shutil.ignore_patterns("__pycache__"))
    kern = DEST / "src" / "dctadjust" / "kernels"
    core = HERE / "_ref" / f"_fastcore{sysconfig.get_config_var('EXT_SUFFIX')}"
    if core.exists():
        shutil.copy2(core, kern / core.name)
    (kern / "_b200.py").write_text(stub_source())
    init = kern / "__init__.py"
    init.write_text(patch_selector(init.read_text()))
    print(f"reference package + b200 stub installed in {DEST.relative_to(ROOT)}", file=sys.stderr)


if __name__ == "__main__":
    main()
