"""Host chunk store with a residency ledger (simulates FPDT's pinned host cache).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

P:L219 "we cache k_i, v_i to the host memory"; "at any given time,
only one set of chunks k_i, v_i is placed on GPU's HBM"; "we
offload q_i, k_i, v_i to the host memory once they are done"; "we mark
them as free memory".  Semantics follow SPEC offload-store:
capacity error, fetch of an absent key errors, checkout high-water mark.
"""
from __future__ import annotations

import numpy as np


class StoreError(RuntimeError):
    pass


class ChunkStore:
    def __init__(self, capacity_bytes: int | None = None):
        self.capacity = capacity_bytes
        self.resident: dict = {}
        self.checked_out: set = set()
        self.bytes_offloaded = 0
        self.bytes_fetched = 0
        self.fetch_count = 0
        self.highwater = 0

    def used(self) -> int:
        return sum(v.nbytes for v in self.resident.values())

    def offload(self, key, chunk: np.ndarray) -> None:
        if key in self.resident:
            raise StoreError(f"duplicate key {key}")
        if self.capacity is not None and self.used() + chunk.nbytes > self.capacity:
            raise StoreError("host capacity exceeded")
        self.resident[key] = np.array(chunk, copy=True)
        self.bytes_offloaded += chunk.nbytes

    def update(self, key, chunk: np.ndarray) -> None:
        """Write back an accumulator (e.g. the dq partial of P:L365) under an existing key."""
        if key not in self.resident:
            raise StoreError(f"missing key {key}")
        self.resident[key] = np.array(chunk, copy=True)
        self.bytes_offloaded += chunk.nbytes

    def fetch(self, key) -> np.ndarray:
        if key not in self.resident:
            raise StoreError(f"missing key {key}")
        self.checked_out.add(key)
        self.highwater = max(self.highwater, len(self.checked_out))
        self.bytes_fetched += self.resident[key].nbytes
        self.fetch_count += 1
        return np.array(self.resident[key], copy=True)

    def release(self, key) -> None:
        if key not in self.checked_out:
            raise StoreError(f"key {key} not checked out")
        self.checked_out.discard(key)

    def free(self, key) -> None:
        if key not in self.resident:
            raise StoreError(f"double free {key}")
        del self.resident[key]
