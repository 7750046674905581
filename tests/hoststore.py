"""Host-only store reading for CPU tests (no GPU): pair arrays + dictionary.

Mirrors storage.load's file handling (/root/reference/pkg/src/gsmat/storage.py:222-271)
without touching the device, so the oracle can run on the same inputs.
"""

from __future__ import annotations

from pathlib import Path

import numpy as np

from paper_1807_07691_b200.dictionary import StoreDictionary
from paper_1807_07691_b200.storage import StatEntry


class HostMatrix:
    def __init__(self, so: np.ndarray, os_: np.ndarray):
        self.so = so
        self.os = os_


class HostStore:
    def __init__(self, directory: Path | str):
        directory = Path(directory)
        self.dictionary = StoreDictionary(directory)
        self.stats = {}
        for raw in (directory / "stats.tsv").read_text().splitlines():
            pid, card, ds, do = (int(x) for x in raw.split("\t"))
            self.stats[pid] = StatEntry(card, ds, do)
        self.matrices = {}
        for pid in self.stats:
            so = np.fromfile(directory / f"p{pid}.so", dtype="<u8").reshape(-1, 2)
            os_ = np.fromfile(directory / f"p{pid}.os", dtype="<u8").reshape(-1, 2)
            self.matrices[pid] = HostMatrix(so, os_)


def plan_for(store, text: str):
    from paper_1807_07691_b200 import frontend

    q = frontend.bind_constants(frontend.parse_query(text), store.dictionary)
    return q, frontend.make_plan(q, store.stats)
