"""The product path has no CPU fallback: without a device, with host tensors or without the
built library it fails loudly instead of computing anything (the oracle is test
infrastructure only)."""
import ast
import os

import pytest
import torch

import paper_1809_07851_b200 as fc
from paper_1809_07851_b200 import _build

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_missing_library_raises(monkeypatch, tmp_path):
    monkeypatch.setattr(fc, "_lib", None)
    monkeypatch.setattr(_build, "LIB", str(tmp_path / "libfastconv.so"))
    with pytest.raises(RuntimeError, match="not built"):
        fc.load()


@pytest.mark.skipif(torch.cuda.is_available(), reason="checks the no-device behaviour")
def test_no_device_plan_raises():
    fc.load()
    with pytest.raises(fc.ConvError):
        fc.Plan(1, 2, 2, 8, 8, 3, "winograd", 2)


def test_host_tensors_rejected():
    x = torch.zeros(1, 2, 8, 8)
    with pytest.raises(ValueError, match="CUDA"):
        fc._check_tensor(x, "x", (1, 2, 8, 8))


def test_product_package_never_imports_the_oracle():
    """Only tests/, __graft_entry__.smoke() and bench.py's baseline legs may touch oracle/."""
    pkg = os.path.join(ROOT, "paper_1809_07851_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if not f.endswith(".py"):
                continue
            tree = ast.parse(open(os.path.join(dirpath, f)).read())
            for node in ast.walk(tree):
                names = []
                if isinstance(node, ast.Import):
                    names = [a.name for a in node.names]
                elif isinstance(node, ast.ImportFrom):
                    names = [node.module or ""]
                assert not any(n == "oracle" or n.startswith("oracle.") for n in names), (f, names)
    for dirpath, _, files in os.walk(os.path.join(pkg, "csrc")):
        for f in files:
            for line in open(os.path.join(dirpath, f), errors="ignore"):
                assert not (line.lstrip().startswith("#include") and "oracle" in line), (f, line)
    assert "oracle" not in open(os.path.join(pkg, "_build.py")).read()  # the library links nothing of it
