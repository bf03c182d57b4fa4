"""Exceptions shared by the ket engine and its callers.

`MemoryBudgetError` mirrors the reference's recoverable budget error
(engine.py:38-44): raised BEFORE any allocation, state left usable.
"""
from __future__ import annotations


class MemoryBudgetError(RuntimeError):
    """A merge/conversion/allocation would exceed the dense amplitude budget."""

    def __init__(self, needed: int, budget: int, detail: str | None = None):
        msg = f"needs {needed} dense amplitudes, budget is {budget}"
        if detail:
            msg += f" ({detail})"
        super().__init__(msg)
        self.needed = needed
        self.budget = budget


class InvariantError(RuntimeError):
    """Internal consistency violation (a bug, not a user error); engine.py:47-48."""


class DeviceError(RuntimeError):
    """A CUDA runtime failure inside libshardcu."""


class DeviceMemoryError(DeviceError, MemoryError):
    """The device itself ran out of memory (cudaMalloc failed).  Distinct from
    MemoryBudgetError: a search that treats a budget error as "p too low"
    (validate.py:292-294) must not mistake a full GPU for it."""
