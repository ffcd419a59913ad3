"""Adapter residency: LoraId -> pool slot mapping with on-demand, asynchronous
host-to-device loading.

The reference models this step only as time: when a request lands on a GPU
whose adapter is not resident, ``Simulator::post_placement`` (core/src/
simulator.cpp:470-479) books ``adapter_load_latency(layers)`` (cost_model.cpp:
91-100: 7 projections x (A + B) x layers over PCIe) and records the completion
time in ``GpuState::adapter_ready_time`` (scheduler.hpp:45).  Here the load is
real: every projection site's A / B for all layers is copied from pinned host
memory into a free (or least-recently-used) slot of the device pools on a
dedicated copy stream, and the completion time becomes a CUDA event the compute
stream waits on before the first SGMV launch that reads the slot.  The SGMV
kernels only ever see slot indices and the pools' device pointer tables, so a
load never rebuilds a table or touches a kernel argument.

:class:`SlotTable` is the pure bookkeeping (LRU over slots, pinning of slots in
use by the current step) and is unit-tested on CPU; :class:`AdapterStore` adds the
pools, pinned staging and events.
"""
from __future__ import annotations

from collections import OrderedDict

import torch

from .sgmv import AdapterPool


class SlotTable:
    """LoraId -> slot with least-recently-used eviction.

    ``acquire(lora_id)`` returns ``(slot, needs_load)``; slots listed in ``pinned``
    (those the in-flight step reads) are never evicted.  Deterministic: free slots
    are handed out in ascending order, eviction takes the least recently acquired.
    """

    def __init__(self, num_slots: int):
        if num_slots < 1:
            raise ValueError("need at least one slot")
        self.num_slots = num_slots
        self._lru: OrderedDict[int, int] = OrderedDict()  # lora_id -> slot, oldest first
        self._free = list(range(num_slots))

    def slot_of(self, lora_id: int) -> int | None:
        return self._lru.get(lora_id)

    def resident(self) -> dict[int, int]:
        return dict(self._lru)

    def acquire(self, lora_id: int, pinned: set[int] | frozenset[int] = frozenset()) -> tuple[int, bool]:
        if lora_id in self._lru:
            self._lru.move_to_end(lora_id)
            return self._lru[lora_id], False
        if self._free:
            slot = self._free.pop(0)
        else:
            victim = next((lid for lid, s in self._lru.items() if s not in pinned), None)
            if victim is None:
                raise RuntimeError("all adapter slots are pinned by the current step")
            slot = self._lru.pop(victim)
        self._lru[lora_id] = slot
        return slot, True

    def release(self, lora_id: int) -> None:
        slot = self._lru.pop(lora_id, None)
        if slot is not None:
            self._free.append(slot)
            self._free.sort()


class AdapterStore:
    """Device pools for several projection sites plus on-demand adapter loading.

    ``sites`` lists ``(h_in, h_out)`` per projection site (Llama: q, k, v, o,
    gate, up, down); every site has its own :class:`AdapterPool` with the same
    slot numbering, so one slot index serves all sites of an adapter.
    """

    def __init__(self, sites, num_slots: int, num_layers: int, rank: int, dtype=torch.float16,
                 device: str | torch.device = "cuda"):
        self.pools = [AdapterPool(num_slots, num_layers, hi, ho, rank, dtype, device=device) for hi, ho in sites]
        self.slots = SlotTable(num_slots)
        self.copy_stream = torch.cuda.Stream(device=device)
        self._ready: dict[int, torch.cuda.Event] = {}

    @property
    def bytes_per_adapter(self) -> int:
        return sum(p.slot_bytes_per_layer * p.num_layers for p in self.pools)

    def load(self, lora_id: int, weights, pinned_slots=frozenset()) -> int:
        """Make ``lora_id`` resident; returns its slot.

        ``weights[i] = (A [layers, h_in, r], B [layers, r, h_out])`` for site i, host
        tensors (pinned for a truly asynchronous copy).  A resident adapter is not
        reloaded.  The copy is queued on ``copy_stream``; call :meth:`wait` on the
        compute stream before launching on the slot.
        """
        slot, needs = self.slots.acquire(lora_id, pinned_slots)
        if not needs:
            return slot
        prev = self._ready.get(slot)
        with torch.cuda.stream(self.copy_stream):
            if prev is not None:  # launches that read the evicted adapter must be done
                self.copy_stream.wait_event(prev)
            for pool, (a, b) in zip(self.pools, weights):
                pool.a[slot].copy_(a, non_blocking=True)
                pool.b[slot].copy_(b, non_blocking=True)
            ev = torch.cuda.Event()
            ev.record(self.copy_stream)
        self._ready[slot] = ev
        return slot

    def wait(self, slots, stream: torch.cuda.Stream | None = None) -> None:
        """Make ``stream`` (default: current) wait for the loads of ``slots``."""
        st = stream or torch.cuda.current_stream()
        for s in set(int(v) for v in slots):
            ev = self._ready.get(s)
            if ev is not None:
                st.wait_event(ev)

    def mark_used(self, slots, stream: torch.cuda.Stream | None = None) -> None:
        """Record that ``stream`` reads ``slots`` from now on: a later eviction of one of
        them waits for this point before overwriting the slot."""
        st = stream or torch.cuda.current_stream()
        for s in set(int(v) for v in slots):
            ev = torch.cuda.Event()
            ev.record(st)
            self._ready[s] = ev


__all__ = ["SlotTable", "AdapterStore"]
