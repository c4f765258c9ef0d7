"""Event trace of real GPU rounds in the reference's schema.

The reference's simulators emit an EventTrace (pipeline.hpp:14-30) serialised by
trace_csv / trace_json (trace_io.cpp:58-105): events (time_sec, resource, kind,
micro_batch, slot) with resource "ssm<j>" or "llm" and kind spec_start / spec_end /
verify_start / verify_end, plus totals llm_busy_sec, llm_idle_sec, accepted_tokens.
Here the times are measured: each spin_round's CUDA events give the per-SSM draft
ends (spin_last_round_trace), the verify start (draft_ms) and the verify end
(round_ms); rounds are laid end to end on the device timeline. One micro-batch per
SSM (micro_batch 0): the verifier is weight-streaming, so splitting it would
re-read the target weights per micro-batch.
"""
from __future__ import annotations

import ctypes as C
import json

import numpy as np

from . import _lib


def _fmt(x: float) -> str:
    return repr(float(x))


class RoundTrace:
    def __init__(self):
        self.events: list[dict] = []
        self.t = 0.0  # device seconds at the start of the next round
        self.llm_busy = 0.0
        self.llm_idle = 0.0
        self.accepted = 0
        self.slot = 0

    def record(self, engine, ssm_of, out: dict) -> None:
        """Append the events of the round `out` (Engine.round) just run on `engine`."""
        m = len(engine.ssms)
        ends = np.zeros(m, np.float32)
        _lib.check(engine.lib.spin_last_round_trace(engine.ctx, ends.ctypes.data_as(_lib.P_F32), m))
        ssm_of = np.asarray(ssm_of)
        t0 = self.t
        for j in range(m):
            if ends[j] < 0 or not (ssm_of == j).any():
                continue
            self.events.append({"time_sec": t0, "resource": f"ssm{j}", "kind": "spec_start", "micro_batch": 0,
                                "slot": self.slot})
            self.events.append({"time_sec": t0 + float(ends[j]) / 1e3, "resource": f"ssm{j}", "kind": "spec_end",
                                "micro_batch": 0, "slot": self.slot})
        v0, v1 = t0 + float(out["draft_ms"]) / 1e3, t0 + float(out["round_ms"]) / 1e3
        self.events.append({"time_sec": v0, "resource": "llm", "kind": "verify_start", "micro_batch": 0,
                            "slot": self.slot})
        self.events.append({"time_sec": v1, "resource": "llm", "kind": "verify_end", "micro_batch": 0,
                            "slot": self.slot})
        self.llm_busy += v1 - v0
        self.llm_idle += v0 - t0
        # accepted + bonus per served request: EventTrace.accepted_tokens sums
        # apply_outcome() (pipeline.cpp:26-35), which counts the bonus token
        served = ssm_of >= 0
        self.accepted += int(np.asarray(out["accepted"])[served].sum()) + int(served.sum())
        self.t = v1
        self.slot += 1

    def csv(self) -> str:
        """trace_csv (trace_io.cpp:58-66)."""
        rows = ["time_sec,resource,kind,micro_batch,slot"]
        for e in self.events:
            rows.append(f"{_fmt(e['time_sec'])},{e['resource']},{e['kind']},{e['micro_batch']},{e['slot']}")
        return "\n".join(rows) + "\n"

    def json(self) -> str:
        """trace_json (trace_io.cpp:68-82)."""
        doc = {"events": self.events,
               "totals": {"llm_busy_sec": self.llm_busy, "llm_idle_sec": self.llm_idle,
                          "accepted_tokens": self.accepted}}
        return json.dumps(doc, indent=2) + "\n"
