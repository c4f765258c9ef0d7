"""Real-round event trace in the reference schema, checked with the invariants of
the reference's pipeline tests (test_pipeline.cpp:191-232): the verifier is
exclusive (verify intervals do not overlap), causal (a slot's verify starts after
every SSM of that slot finished drafting), and busy + idle spans the makespan."""
import csv
import io
import json

import numpy as np
import pytest

from paper_2503_15921_b200.models import TINY_SSMS, TINY_TARGET, Engine, synthetic_prompts
from paper_2503_15921_b200.trace import RoundTrace

pytestmark = pytest.mark.gpu


def test_trace_schema_and_invariants():
    B = 8
    eng = Engine(TINY_TARGET, TINY_SSMS, max_requests=B, max_ctx=256, window=4)
    eng.prefill(range(B), synthetic_prompts(B, 16, 64, TINY_TARGET.vocab, 99))
    slots = np.arange(B, dtype=np.int32)
    tr = RoundTrace()
    emitted = 0
    for r in range(4):
        assign = np.array([(i + r) % 2 for i in range(B)], np.int32)
        if r == 3:
            assign[:4] = -1  # idle requests
        out = eng.round(slots, assign)
        tr.record(eng, assign, out)
        emitted += int(out["accepted"][assign >= 0].sum()) + int((assign >= 0).sum())
    eng.close()
    rows = list(csv.DictReader(io.StringIO(tr.csv())))
    assert list(rows[0].keys()) == ["time_sec", "resource", "kind", "micro_batch", "slot"]
    doc = json.loads(tr.json())
    assert set(doc["totals"]) == {"llm_busy_sec", "llm_idle_sec", "accepted_tokens"}
    verify = [(float(a["time_sec"]), float(b["time_sec"]), int(a["slot"]))
              for a, b in zip([r for r in rows if r["kind"] == "verify_start"],
                              [r for r in rows if r["kind"] == "verify_end"])]
    for (s0, e0, _), (s1, e1, _) in zip(verify, verify[1:]):
        assert s0 <= e0 <= s1 <= e1  # exclusive verifier, slots in order
    for s0, _, slot in verify:
        ends = [float(r["time_sec"]) for r in rows if r["kind"] == "spec_end" and int(r["slot"]) == slot]
        assert ends and max(ends) <= s0 + 1e-9  # causality
    makespan = verify[-1][1]
    assert abs(doc["totals"]["llm_busy_sec"] + doc["totals"]["llm_idle_sec"] - makespan) < 1e-6
    assert doc["totals"]["accepted_tokens"] == emitted  # accepted + bonus (pipeline.cpp:26-35)
