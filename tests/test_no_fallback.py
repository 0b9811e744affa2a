"""The product path has no CPU fallback and never touches the oracle (CPU tests).

* using the package from a copy without ``libnsdgt.so`` raises ImportError (the package
  loads the library lazily, on the first API name, so that the build module runs first);
* no source of the package (Python, CUDA, C++) refers to ``oracle`` -- the oracle is test
  infrastructure, importable only by tests/, smoke() and bench.py's CPU legs.
"""
import os
import pathlib
import shutil
import subprocess
import sys

ROOT = pathlib.Path(__file__).resolve().parents[1]
PKG = ROOT / "paper_1307_4569_b200"


def test_import_without_library_fails_loudly(tmp_path):
    dst = tmp_path / "paper_1307_4569_b200"
    shutil.copytree(PKG, dst, ignore=shutil.ignore_patterns("*.so", "__pycache__", "csrc"))
    assert not any(dst.glob("*.so"))
    code = "import paper_1307_4569_b200 as m; m.Plan"
    env = dict(os.environ, PYTHONPATH=str(tmp_path))
    r = subprocess.run([sys.executable, "-c", code], cwd=tmp_path, env=env, capture_output=True, text=True)
    assert r.returncode != 0
    assert "ImportError" in r.stderr and "no CPU fallback" in r.stderr


def test_package_never_refers_to_the_oracle():
    offenders = []
    for p in PKG.rglob("*"):
        if p.suffix in (".py", ".cu", ".cuh", ".cpp", ".hpp", ".h") and "oracle" in p.read_text().lower():
            offenders.append(str(p.relative_to(ROOT)))
    assert not offenders, offenders
