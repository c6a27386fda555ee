"""The reference's own test file (pkg/tests/test_qmath.py), run UNCHANGED against this
package: ``qnmt`` / ``qnmt.qmath`` / ``qnmt.errors`` are aliased to the facade in a child
pytest process, so every ``from qnmt.qmath import ...`` of that file binds the B200 path
(consequence 1).

The file is not part of this repository: ``__graft_entry__.build()`` copies the reference's
``pkg/tests`` next to the reference install (``baseline/_ref/_tests``, git-ignored, travels to
the GPU box).  Without that copy (and without /root/reference) the test is skipped.
"""

import os
import subprocess
import sys
import textwrap

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CANDIDATES = [os.path.join(ROOT, "baseline", "_ref", "_tests"), "/root/reference/pkg/tests"]

ALIAS_PLUGIN = textwrap.dedent("""
    import sys
    sys.path.insert(0, {root!r})
    import paper_1804_05038_b200 as pb
    from paper_1804_05038_b200 import errors, qmath
    sys.modules["qnmt"] = pb
    sys.modules["qnmt.qmath"] = qmath
    sys.modules["qnmt.errors"] = errors
""")


def _ref_tests():
    for d in CANDIDATES:
        if os.path.isfile(os.path.join(d, "test_qmath.py")):
            return d
    return None


@pytest.mark.gpu
def test_reference_test_qmath_passes_unchanged_on_the_facade(tmp_path):
    d = _ref_tests()
    if d is None:
        pytest.skip("reference test files not available (baseline/_ref/_tests is made by build())")
    plugin = tmp_path / "qnmt_alias_plugin.py"
    plugin.write_text(ALIAS_PLUGIN.format(root=ROOT))
    env = dict(os.environ, PYTHONPATH=str(tmp_path) + os.pathsep + os.environ.get("PYTHONPATH", ""))
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-p", "qnmt_alias_plugin", "-p", "no:cacheprovider",
                        "--rootdir", str(tmp_path), "-c", os.devnull, os.path.join(d, "test_qmath.py")],
                       capture_output=True, text=True, env=env, cwd=str(tmp_path), timeout=900)
    tail = (r.stdout + r.stderr)[-3000:]
    assert r.returncode == 0, tail
    assert " passed" in r.stdout and "failed" not in r.stdout, tail


def test_alias_plugin_targets_exist():
    """CPU: the names the reference test file imports exist on the facade."""
    from paper_1804_05038_b200 import errors, qmath
    for name in ("QuantizedMatrix", "dequantize", "gemm_f32", "gemm_f32_blocked", "qgemm", "qgemm_panel",
                 "quantize", "INT32_SAFE_K"):
        assert hasattr(qmath, name), name
    for name in ("InvalidInputError", "ShapeError"):
        assert hasattr(errors, name), name
