"""Adapter residency (paper_2310_18547_b200/adapters.py): LRU slot bookkeeping on
CPU, and on the GPU asynchronous loads feeding SGMV launches through the same
slot indices (reference: post_placement, simulator.cpp:470-479;
adapter_ready_time, scheduler.hpp:45)."""
from __future__ import annotations

import numpy as np
import pytest
import torch

from paper_2310_18547_b200.adapters import SlotTable
from tests._util import TOL, oracle, row_norm_err


def test_slot_table_lru_and_pinning():
    t = SlotTable(3)
    assert t.acquire(10) == (0, True)
    assert t.acquire(11) == (1, True)
    assert t.acquire(10) == (0, False)          # resident: no load, becomes most recent
    assert t.acquire(12) == (2, True)
    assert t.acquire(13) == (1, True)           # evicts 11 (least recent)
    assert t.slot_of(11) is None and t.slot_of(13) == 1
    assert t.acquire(14, pinned={0}) == (2, True)  # 10 (slot 0) pinned -> evict 12 (slot 2)
    with pytest.raises(RuntimeError):
        t.acquire(15, pinned={0, 1, 2})
    t.release(10)
    assert t.acquire(16) == (0, True)           # released slot is reused first
    with pytest.raises(ValueError):
        SlotTable(0)


@pytest.mark.gpu
def test_async_loads_feed_sgmv_and_survive_eviction():
    import paper_2310_18547_b200 as lsg
    from paper_2310_18547_b200.adapters import AdapterStore
    assert torch.cuda.is_available()
    h, r, layers = 4096, 16, 2
    sites = [(h, h), (h, h)]
    store = AdapterStore(sites, num_slots=2, num_layers=layers, rank=r, dtype=torch.float16)
    rng = oracle().rng(77)
    host = {}
    for lid in (100, 200, 300):
        w = []
        for _ in sites:
            a = torch.tensor(rng.fill_pm1(layers * h * r).reshape(layers, h, r)).half().pin_memory()
            b = torch.tensor(rng.fill_pm1(layers * r * h).reshape(layers, r, h)).half().pin_memory()
            w.append((a, b))
        host[lid] = w
    x = torch.tensor(rng.fill_pm1(3 * h).reshape(3, h)).half().cuda()
    seg_starts = torch.tensor([0, 2, 3], dtype=torch.int32, device="cuda")

    def run(lids, layer, site):
        slots = [store.load(l, host[l], pinned_slots=set()) for l in lids]
        store.wait(slots)
        y = torch.zeros(3, h, dtype=torch.float16, device="cuda")
        lsg.sgmv(y, x, store.pools[site], seg_starts, torch.tensor(slots, dtype=torch.int32, device="cuda"), layer)
        store.mark_used(slots)
        torch.cuda.synchronize()
        A = np.stack([host[l][site][0][layer].double().numpy() for l in lids])
        B = np.stack([host[l][site][1][layer].double().numpy() for l in lids])
        ref = oracle().lora_addon(x.double().cpu().numpy(), np.array([0, 2, 3], dtype=np.uint64), A, B)
        return row_norm_err(y.double().cpu().numpy(), ref)

    assert run([100, 200], 1, 0) <= TOL["float16"]
    assert run([300, 200], 0, 1) <= TOL["float16"]   # 300 evicts 100
    assert store.slots.slot_of(100) is None
    assert run([100, 300], 1, 1) <= TOL["float16"]   # 100 reloaded over 200's slot
