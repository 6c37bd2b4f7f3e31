"""The C-ABI library loads and exports every symbol include/taper.h declares (CPU-only:
no compute calls), and the host-side validation paths that need no device."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    src = open(os.path.join(ROOT, "include", "taper.h")).read()
    return sorted(set(re.findall(r"TAPER_API\s+[\w\s\*]+?\b(taper_\w+)\s*\(", src)))


def test_header_declares_the_boundary():
    names = _declared()
    for n in ("taper_admit", "taper_decode_attention", "taper_build_work", "taper_workspace_size",
              "taper_status_string"):
        assert n in names


def test_library_exports_every_declared_symbol():
    from paper_2605_06914_b200 import build
    lib_path = build.build()
    lib = ctypes.CDLL(lib_path)
    for n in _declared():
        assert hasattr(lib, n), n
    from paper_2605_06914_b200 import taper as T
    assert set(T.EXPORTS) == set(_declared())


def test_host_validation_without_gpu():
    from paper_2605_06914_b200 import taper as T
    assert T.taper_workspace_size(64, 192, 8, 768) > 768 * 8 * 8 * 129 * 4
    with pytest.raises(T.TaperError):
        T.taper_workspace_size(5000, 10, 8, 1)
    with pytest.raises(T.TaperError):
        T.taper_workspace_size(10, 10, 9, 1)
    assert "monotone" in T.taper_status_string(-3)
    assert "precision" in T.taper_status_string(4)
    # a 3-request batch splits at the 1024-token floor: 5 chunks x 3 ready branches + 1 x 1
    # + 0 x 2, plus one local item per branch with local tokens (65, 1, 2, 3 -> 4 items of
    # <= 16 x 64 tokens)
    assert T.max_chunk_slots([4097, 1, 0], [0, 3, 4, 6], [0, 65, 1, 0, 2, 3], h_local=8) == 15 + 1 + 0 + 4
    # taper_chunk_tokens(Lsh, h, R) (include/taper.h): clamp(Lsh h R / 512, 1024, 4096) --
    # C2 (R = 64, 4k prefixes): 1024 at h <= 2, 2048 at h = 4, 4096 at h = 8; C3 (R = 32) 24k
    # prefix: 1536 at h = 1, 4096 at h >= 4; C5 (R = 256) 9k prefix: 4096 even at h = 1.
    # Probed as the chunk count of request 0 (one slot; the others are empty).
    def chunks(lsh, h, R=1):
        return T.max_chunk_slots([lsh] + [0] * (R - 1), list(range(R + 1)), [0] * R, h_local=h)
    assert [chunks(4096, h, 64) for h in (1, 2, 4, 8)] == [4, 4, 2, 1]
    assert [chunks(24576, h, 32) for h in (1, 2, 4, 8)] == [16, 8, 6, 6]
    assert chunks(9216, 1, 256) == 3
    assert chunks(100, 8) == 1 and chunks(1025, 1) == 2 and chunks(0, 1) == 0
    # local segments count per segment; bad CSR is an argument error
    assert T.max_chunk_slots([0], [0, 1], [1030], [1024, 6], h_local=8,
                             slot_seg_off=[0, 2]) == 2
    with pytest.raises(T.TaperError):
        T.max_chunk_slots([5], [0, 2], [1], h_local=8)
    assert T.max_chunk_slots([4097, 1, 0], [0, 3, 4, 6], [0, 65, 1, 0, 2, 3]) == 15 + 1 + 0 + 4


def test_gather_and_ipc_host_validation_without_gpu():
    """The fused-gather / IPC entry points (include/taper.h) reject bad arguments on the host
    before touching the device."""
    import ctypes
    from paper_2605_06914_b200 import taper as T
    lib = T._lib
    # rank outside the world, world not a power of two up to 8, null flags
    for world, rank in ((2, 2), (3, 0), (2, -1)):
        g = T.Gather(world, 0, [0] * world, [0] * world)
        g._c.rank = rank
        assert lib.taper_gather_wait(ctypes.byref(g.c()), None) == T.TAPER_OK - 1  # TAPER_ERR_ARG
    assert lib.taper_decode_attention_gather(None, None, None, None, None, None, 1.0, None, 0, None) == -1
    assert lib.taper_ipc_handle(None, None, None) == -1
    assert lib.taper_ipc_open(None, 0, None) == -1
    assert lib.taper_ipc_close(None, 0) == -1
