"""Stage the reference package as TEST-ONLY data for the GPU box.

CHECKER INFRASTRUCTURE, like ``oracle/_ref``'s compiled outputs: run by
``__graft_entry__.build()`` in the build container (where ``/root/reference``
exists).  It zips the reference's Python sources and its unit tests, unchanged,
into ``oracle/_ref/recycg_ref.zip`` (git-ignored, not gpurun-ignored), so
``tests/test_gpu_reference_bridge.py`` can run the reference's own
``test_solver.py`` / ``test_ritz.py`` / ``test_recycle.py`` on the GPU box with
the reference's seams rebound to the B200 path (``paper_1301_7530_b200.bridge``).
Nothing in the product, ``bench.py`` or ``smoke()`` reads this archive.
"""
from __future__ import annotations

import zipfile
from pathlib import Path

REF = Path("/root/reference/pkg")
OUT = Path(__file__).resolve().parent / "_ref" / "recycg_ref.zip"


def stage(out=OUT, ref=REF):
    if not (ref / "src" / "recycg").is_dir():
        return None
    out.parent.mkdir(parents=True, exist_ok=True)
    tmp = out.with_suffix(".tmp")
    files = [(p, f"src/recycg/{p.name}") for p in sorted((ref / "src" / "recycg").glob("*.py"))]
    files += [(p, f"tests/{p.name}") for p in sorted((ref / "tests").glob("*.py"))]
    files += [(p, f"tests/fixtures/{p.name}") for p in sorted((ref / "tests" / "fixtures").glob("*"))]
    with zipfile.ZipFile(tmp, "w", zipfile.ZIP_DEFLATED) as z:
        for p, arc in files:
            z.writestr(zipfile.ZipInfo(arc, date_time=(2020, 1, 1, 0, 0, 0)), p.read_bytes())
    tmp.replace(out)
    return out


if __name__ == "__main__":
    print(stage())
