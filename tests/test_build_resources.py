"""Build guard (CPU): the fused kernel's resource budget.  Two CTAs per SM need <= 128 registers per
thread; measured on the B200, a larger stack frame (spilled / out-of-line code) slows every launch
(CTAs start microseconds late), so the frame is capped at what the fast build uses."""
import os
import re
import shutil
import subprocess

import pytest

LIB = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                   "paper_2602_01518_b200", "lib", "libqrita_b200.so")


@pytest.mark.skipif(not os.path.exists(LIB) or shutil.which("cuobjdump") is None,
                    reason="library not built or cuobjdump missing")
def test_fused_kernel_budget():
    out = subprocess.run(["cuobjdump", "-res-usage", LIB], capture_output=True, text=True).stdout
    blocks = re.findall(r"Function (\S+):\s*\n\s*REG:(\d+) STACK:(\d+)", out)
    fused = {name: (int(r), int(st)) for name, r, st in blocks if "qrita_fused" in name}
    assert fused, "qrita_fused not found in the library"
    for name, (reg, stack) in fused.items():
        assert reg <= 128, (name, reg)
        assert stack <= 1200, (name, stack)
