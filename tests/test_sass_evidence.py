"""The built library contains the Blackwell instructions DESIGN.md claims (CPU test:
cuobjdump -sass of libparareal.so): TMA tensor loads (UTMALDG) and mbarrier ops (SYNCS)
in the persistent F and G kernels; tcgen05.ld / tcgen05.st (LDTM / STTM) and
tcgen05.alloc in the TMEM hand-off kernels (PR_FTILE=23, the default F for n >= 256); no
legacy tensor-core or Hopper instructions anywhere (HMMA, HGMMA)."""
import os
import shutil
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "tools"))
LIB = os.path.join(ROOT, "paper_1409_8563_b200", "libparareal.so")

pytestmark = pytest.mark.skipif(not shutil.which("cuobjdump") or not os.path.exists(LIB),
                                reason="needs cuobjdump and the built library")


@pytest.fixture(scope="module")
def mix():
    import sass_mix
    return sass_mix.mix(LIB)


def kernels(mix, *parts):
    return {f: c for f, c in mix.items() if all(p in f for p in parts)}


def test_default_kernels_use_tma_and_mbarriers(mix):
    default = kernels(mix, "fused_persist_kernel", "ELi9ELi0ELi0EE")  # variant 14 (n < 256)
    assert len(default) >= 2
    for f, c in default.items():
        assert c["UTMALDG"] >= 1 and c["SYNCS"] >= 10 and c["DFMA"] > 500, f
    coarse = kernels(mix, "coarse_persist_kernel")
    assert coarse and all(c["UTMALDG"] >= 1 for c in coarse.values())


def test_tmem_variant_uses_tcgen05(mix):
    tm = kernels(mix, "fused_persist_kernel", "ELi9ELi1E")  # TM = 1 (variant 23, n >= 256)
    assert len(tm) >= 2
    for f, c in tm.items():
        assert c["LDTM"] >= 1 and c["STTM"] >= 1 and c["UTCATOMSWS"] >= 1, f
        assert c["UTMALDG"] >= 1 and c["SYNCS"] >= 10 and c["DFMA"] > 500, f


def test_no_legacy_tensor_core_or_hopper_instructions(mix):
    for f, c in mix.items():
        assert not (c["HMMA"] or c["HGMMA"] or c["QGMMA"]), f
