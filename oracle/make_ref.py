"""TEST INFRASTRUCTURE -- vendors the reference for parity level 4 and the
reference benchmark arm.  Never imported by the product package.

The reference (arXiv 1703.02438 re-implementation, package ``nmk``) is pure
Python: it has no build step, so "building" it for oracle/_ref means copying
its package and its own test files out of the read-only reference tree:

    /root/reference/pkg/src/nmk/*.py   -> oracle/_ref/nmk/
    /root/reference/pkg/tests/*.py     -> oracle/_ref/tests/

oracle/_ref/ is git-ignored (reference sources never enter this repo's
history) but NOT gpurun-ignored, so it travels to the GPU box with the
snapshot, like a compiled oracle/_ref .so would.  A MANIFEST.json records the
SHA-256 of every copied file.  ``__graft_entry__.build()`` runs this when
/root/reference is present; on the GPU box only the copied tree is used.

    python oracle/make_ref.py [--src /root/reference/pkg] [--dst oracle/_ref]
"""

from __future__ import annotations

import argparse
import hashlib
import json
import os
import shutil

HERE = os.path.dirname(os.path.abspath(__file__))
DEFAULT_SRC = "/root/reference/pkg"
DEFAULT_DST = os.path.join(HERE, "_ref")


def build(src: str = DEFAULT_SRC, dst: str = DEFAULT_DST) -> dict:
    pkg = os.path.join(src, "src", "nmk")
    tests = os.path.join(src, "tests")
    if not os.path.isdir(pkg):
        raise FileNotFoundError(f"reference package not found at {pkg}")
    manifest = {"source": src, "files": {}}
    for sub, from_dir in (("nmk", pkg), ("tests", tests)):
        out = os.path.join(dst, sub)
        if os.path.isdir(out):
            shutil.rmtree(out)
        os.makedirs(out)
        for name in sorted(os.listdir(from_dir)):
            if not name.endswith(".py"):
                continue
            with open(os.path.join(from_dir, name), "rb") as f:
                data = f.read()
            with open(os.path.join(out, name), "wb") as f:
                f.write(data)
            manifest["files"][f"{sub}/{name}"] = hashlib.sha256(data).hexdigest()
    with open(os.path.join(dst, "MANIFEST.json"), "w") as f:
        json.dump(manifest, f, indent=1, sort_keys=True)
    return manifest


def present(dst: str = DEFAULT_DST) -> bool:
    return os.path.exists(os.path.join(dst, "nmk", "pipeline.py"))


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--src", default=DEFAULT_SRC)
    ap.add_argument("--dst", default=DEFAULT_DST)
    a = ap.parse_args()
    m = build(a.src, a.dst)
    print(f"oracle/_ref: {len(m['files'])} files from {a.src}")
