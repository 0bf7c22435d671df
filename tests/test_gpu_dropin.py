"""The drop-in, proven inside the reference.

A scratch copy of the unmodified reference package (oracle/_ref, built by
oracle/build_ref.sh) gets exactly the binding INTEGRATION.md s2 tells a
maintainer to add -- `whff/_kernels_b200.py` re-exporting this package's
plugin module and the `WHFF_BACKEND=b200` branch in `whff/backend.py`
(reference backend.py:20-46) -- and then the reference's OWN test files run
against it with `WHFF_BACKEND=b200`:

  * test_codec.py, test_mpgemv.py: every codec / GEMV call of the reference
    goes through the B200 kernels (the plugin contract, backend.py:36-46);
  * test_backends.py with its second backend switched from "compiled" to
    "b200": the reference's own cross-backend bit-identity checks (GEMV
    policies x reduction shapes, codec bytes in every mode, cross decode;
    tests/test_backends.py:19-64) compare the numpy backend with ours.

The reference tests are copied next to the build (oracle/_ref/_reference_tests,
git-ignored); the test skips when that build is absent.
"""

import os
import re
import shutil
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(ROOT, "oracle", "_ref")

KERNELS_B200 = '''"""B200 kernels for the whff plugin contract (backend.py:36-46)."""
from paper_1902_08018_b200.backend import NAME, gemv_kernel, encode_blocks, decode_blocks  # noqa: F401
'''


def patch_backend(src):
    """INTEGRATION.md s2, applied to the reference's backend.py."""
    src = src.replace(
        "except ImportError:  # extension not built\n    _compiled = None\n",
        "except ImportError:  # extension not built\n    _compiled = None\n"
        "\ntry:\n    from . import _kernels_b200 as _b200\nexcept ImportError:\n    _b200 = None\n", 1)
    src = src.replace(
        "elif _forced:\n",
        "elif _forced == \"b200\":\n"
        "    if _b200 is None:\n"
        "        raise ImportError(\"WHFF_BACKEND=b200 but paper_1902_08018_b200 is not importable\")\n"
        "    kernels = _b200\n"
        "elif _forced:\n", 1)
    src = src.replace(
        "        out[\"compiled\"] = _compiled\n    return out\n",
        "        out[\"compiled\"] = _compiled\n    if _b200 is not None:\n"
        "        out[\"b200\"] = _b200\n    return out\n", 1)
    assert src.count("_b200") >= 5, "reference backend.py changed shape; INTEGRATION.md s2 needs updating"
    return src


@pytest.fixture(scope="module")
def patched_reference(tmp_path_factory):
    tests = os.path.join(REF, "_reference_tests")
    if not (os.path.isdir(os.path.join(REF, "whff")) and os.path.isdir(tests)):
        pytest.skip("oracle/_ref (the reference build and its tests) not present")
    root = tmp_path_factory.mktemp("ref_b200")
    shutil.copytree(os.path.join(REF, "whff"), root / "whff")
    (root / "whff" / "_kernels_b200.py").write_text(KERNELS_B200)
    be = root / "whff" / "backend.py"
    be.write_text(patch_backend(be.read_text()))
    shutil.copytree(tests, root / "tests")
    tb = root / "tests" / "test_backends.py"
    src = tb.read_text()
    # the reference's cross-backend checks, second backend = the B200 plugin
    src = re.sub(r'"compiled"', '"b200"', src)
    tb.write_text(src)
    return root


def run_reference_tests(root, files):
    env = dict(os.environ)
    env["PYTHONPATH"] = os.pathsep.join([str(root), ROOT])
    env["WHFF_BACKEND"] = "b200"
    cmd = [sys.executable, "-m", "pytest", "-q", "-p", "no:cacheprovider", "--rootdir", str(root),
           *[str(root / "tests" / f) for f in files]]
    return subprocess.run(cmd, cwd=str(root), env=env, capture_output=True, text=True, timeout=1200)


def test_reference_selects_b200_backend(patched_reference):
    env = dict(os.environ, PYTHONPATH=os.pathsep.join([str(patched_reference), ROOT]), WHFF_BACKEND="b200")
    out = subprocess.run([sys.executable, "-c",
                          "import whff, whff.backend as b; print(whff.BACKEND_NAME, sorted(b.available_backends()))"],
                         env=env, capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr
    assert out.stdout.split()[0] == "b200", out.stdout


@pytest.mark.parametrize("files", [["test_codec.py", "test_mpgemv.py"], ["test_backends.py"]])
def test_reference_suite_on_b200(patched_reference, files):
    r = run_reference_tests(patched_reference, files)
    tail = (r.stdout + r.stderr)[-4000:]
    assert r.returncode == 0, tail
    assert " passed" in r.stdout and " failed" not in r.stdout, tail
