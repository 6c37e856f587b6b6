"""Restatement of the Adaptive Hogbatch controller (test oracle only).

Algorithm 2 of the paper as implemented by the reference
in `policies.py:84-129`, plus the proportional learning-rate rule
(`policies.py:34-36`) and initial sizes (`policies.py:46-51`).
"""

from __future__ import annotations


def scaled_learning_rate(base_eta, batch_size, reference_batch):
    """eta = base_eta * b / ref_b (policies.py:34-36)."""
    return base_eta * (batch_size / reference_batch)


def initial_batch_size(is_replica, threads, min_batch, max_batch):
    """Replica workers start at max_batch, sharded pools at one example per
    thread clamped to the thresholds (policies.py:46-51)."""
    if is_replica:
        return max_batch
    return min(max(threads, min_batch), max_batch)


class OracleAdaptive:
    """State of AdaptiveState (policies.py:63-81) with adaptive_update
    (policies.py:84-129)."""

    def __init__(self, alpha=2.0):
        if alpha <= 1.0:
            raise ValueError("alpha must be > 1")
        self.alpha = alpha
        self.slots = {}  # wid -> [batch, min_b, max_b, u, reported_once]
        self.min_updates = 0.0
        self.max_updates = 0.0

    def register(self, wid, batch, min_b, max_b):
        self.slots[wid] = [batch, min_b, max_b, 0.0, False]
        return batch

    def update(self, wid, reported_u, strict=False):
        slot = self.slots[wid]
        if reported_u < slot[3]:
            raise ValueError(f"update count for {wid} went backwards")
        slot[3] = reported_u
        if not slot[4]:
            slot[4] = True
            return slot[0]
        if strict:
            others = [s[3] for w, s in self.slots.items() if w != wid]
            if not others:
                return slot[0]
            min_u, max_u = min(others), max(others)
        else:
            min_u, max_u = self.min_updates, self.max_updates
        if reported_u < min_u:
            slot[0] = max(int(slot[0] / self.alpha), slot[1])
            if not strict:
                self.min_updates = reported_u
        elif reported_u > max_u:
            slot[0] = min(int(slot[0] * self.alpha), slot[2])
            if not strict:
                self.max_updates = reported_u
        return slot[0]
