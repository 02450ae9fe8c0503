"""Register budgets of the hot kernels in the built library (CPU-only: reads the cubin's
resource table with cuobjdump, no GPU).  The occupancy each kernel was measured at depends on
these counts (K7 is only fast at 40 registers / 6 CTAs per SM -- a loop rewrite that
let ptxas take 52 registers cost 9 %; K6 64 -> 4 CTAs/SM; K8 96 -> 5 CTAs/SM)."""
import os
import re
import shutil
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "paper_2409_06765_b200", "libgsplat_b200.so")

# kernel-name pattern (the default, dense RGB instantiation) -> max registers per thread
BUDGETS = {
    r"k_raster_bwdILb0ELb0ELb0E": 40,
    r"k_raster_fwdILb0ELb0ELb0E": 64,
    r"k_project_bwdILi3ELb0E": 96,
}


def _usage():
    exe = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    if not os.path.exists(LIB) or not os.path.exists(exe):
        pytest.skip("library or cuobjdump not available")
    out = subprocess.run([exe, "--dump-resource-usage", LIB], capture_output=True, text=True).stdout
    regs = {}
    fn = None
    for line in out.splitlines():
        m = re.match(r"\s*Function (\S+):", line)
        if m:
            fn = m.group(1)
            continue
        m = re.search(r"REG:(\d+) STACK:(\d+)", line)
        if m and fn:
            regs[fn] = (int(m.group(1)), int(m.group(2)))
            fn = None
    return regs


@pytest.mark.parametrize("pat,budget", sorted(BUDGETS.items()))
def test_register_budget(pat, budget):
    regs = _usage()
    hits = {f: r for f, r in regs.items() if re.search(pat, f)}
    assert hits, f"no kernel matching {pat} in {LIB}"
    for f, (reg, stack) in hits.items():
        assert reg <= budget, f"{f}: {reg} registers > {budget} (occupancy the kernel was tuned at)"
        assert stack == 0, f"{f}: {stack} bytes of stack (spills)"
