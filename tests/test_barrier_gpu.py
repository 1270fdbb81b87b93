"""The world-barrier protocol with the barriers ON, on one GPU (tests/test_layer_gpu.py's
lockstep emulation disables them).  Separate spinning launches per emulated rank are not
guaranteed to be co-scheduled on one GPU, so the ranks are the CTAs of ONE cooperative
launch (fssdp_barrier_selftest) running the product's world_barrier_warp on the emulated
ranks' real symmetric heaps and flag pads: each round every rank stores a stamp block into
every peer heap, joins the barrier, and checks every block in its own heap.  Any missing
release/acquire ordering shows up as a stale stamp; a lost arrival as the barrier's
30 s trap.  The multi-process path itself: tests/test_dist_gpu.py (>= 2 GPUs)."""

import ctypes as C

import pytest
import torch

from paper_2502_02581_b200 import _native as N
from paper_2502_02581_b200.comm import HeapLayout, emulated_group

pytestmark = pytest.mark.gpu

SELFTEST_BYTES = 2 * 32 * 256 * 4  # FSSDP_SELFTEST_BYTES


@pytest.mark.parametrize("world", [2, 4, 8, 32])
def test_world_barrier_orders_peer_stores(world):
    layout = HeapLayout()
    off = layout.add("selftest", SELFTEST_BYTES)
    groups = emulated_group(layout, world)
    g0 = groups[0]
    errors = torch.zeros(1, dtype=torch.int32, device="cuda")
    stream = C.c_void_p(torch.cuda.current_stream().cuda_stream)
    pb = C.c_void_p(g0.peer_bases.data_ptr())
    flags = layout.offset("flags")
    epoch = 1
    for rounds in (1, 257, 2000):  # epochs keep growing across launches, never reset
        N.call("fssdp_barrier_selftest", pb, flags, off, world, rounds, 5, C.c_uint32(epoch),
               2000 if rounds == 257 else 0, C.c_void_p(errors.data_ptr()), stream)
        epoch += rounds
        torch.cuda.synchronize()
        assert int(errors.item()) == 0, f"{errors.item()} stale words at world {world}"
    # every rank's arrival flag for slot 5 on every heap holds the last epoch
    for r in range(world):
        pad = groups[r].local.tensor(flags, (72, 32), torch.int32)
        assert pad[5, :world].tolist() == [epoch - 1] * world


def test_selftest_detects_a_missing_barrier():
    """Negative control: the same rounds with the barrier skipped (slot -1) and the ranks'
    stores skewed by 2 us per rank must read stale stamps — the check above is live."""
    layout = HeapLayout()
    off = layout.add("selftest", SELFTEST_BYTES)
    g = emulated_group(layout, 8)[0]
    errors = torch.zeros(1, dtype=torch.int32, device="cuda")
    N.call("fssdp_barrier_selftest", C.c_void_p(g.peer_bases.data_ptr()), layout.offset("flags"),
           off, 8, 500, -1, C.c_uint32(1), 2000, C.c_void_p(errors.data_ptr()),
           C.c_void_p(torch.cuda.current_stream().cuda_stream))
    torch.cuda.synchronize()
    assert int(errors.item()) > 0


def test_selftest_rejects_bad_arguments():
    layout = HeapLayout()
    layout.add("selftest", SELFTEST_BYTES)
    g = emulated_group(layout, 2)[0]
    with pytest.raises(Exception):
        N.call("fssdp_barrier_selftest", C.c_void_p(g.peer_bases.data_ptr()),
               layout.offset("flags"), 0, 33, 1, 0, C.c_uint32(1), 0, None,
               C.c_void_p(torch.cuda.current_stream().cuda_stream))
