"""ORACLE build recipe — test infrastructure only.

Two artefacts, both git-ignored and both shipped to the GPU box by gpurun:

* oracle/_build/liboracle_scan.so — the plain-C restatement of the
  reference's nearest-codeword scan (nearest_scan.c), gcc -O3
  -ffp-contract=off exactly like the reference's own build flags
  (/root/reference/pkg/setup.py:22-24).
* oracle/_ref/hqmq/ — the UNMODIFIED reference package, built from its own
  sources by pip (setuptools + Cython, the reference's declared build,
  /root/reference/pkg/pyproject.toml:1-3) from a scratch copy under /tmp
  (the source tree is read-only) with --target oracle/_ref. It is only
  available where /root/reference exists (this build container); on the GPU
  box the prebuilt copy travels with the snapshot. It serves as the
  "reference" CPU baseline in bench.py and as an extra parity witness.

Nothing here is imported by the product package.
"""

from __future__ import annotations

import os
import shutil
import subprocess
import sys
import tempfile

HERE = os.path.dirname(os.path.abspath(__file__))
REF_SRC = "/root/reference/pkg"
REF_DIR = os.path.join(HERE, "_ref")


def build_scan() -> str:
    sys.path.insert(0, HERE)
    try:
        import hqmq_oracle
    finally:
        sys.path.pop(0)
    return hqmq_oracle.build_oracle()


def ref_available() -> bool:
    return os.path.exists(os.path.join(REF_DIR, "hqmq", "__init__.py"))


def build_ref(force: bool = False) -> bool:
    """pip-install the reference into oracle/_ref (no network, no deps)."""
    if ref_available() and not force:
        return True
    if not os.path.isdir(REF_SRC):
        return ref_available()
    with tempfile.TemporaryDirectory() as tmp:
        src = os.path.join(tmp, "pkg")
        shutil.copytree(REF_SRC, src)
        stage = os.path.join(tmp, "target")
        cmd = [sys.executable, "-m", "pip", "install", "--no-index",
               "--no-build-isolation", "--no-deps", "--find-links",
               "/opt/wheelhouse", "--target", stage, src]
        subprocess.check_call(cmd, stdout=subprocess.DEVNULL)
        if os.path.exists(REF_DIR):
            shutil.rmtree(REF_DIR)
        shutil.copytree(stage, REF_DIR)
    return ref_available()


def import_ref():
    """Import the installed reference package as `hqmq` (or None)."""
    if not ref_available():
        return None
    if REF_DIR not in sys.path:
        sys.path.insert(0, REF_DIR)
    import hqmq  # noqa: F401

    return hqmq


if __name__ == "__main__":
    print(build_scan())
    print("reference:", build_ref("--force" in sys.argv))
