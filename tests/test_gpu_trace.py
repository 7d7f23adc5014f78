"""Trace spans and the collective ledger: the records dd_evaluate writes
to a TraceSink / CollectiveLedger (decomp.cpp:285-538, PayloadLayout decomp.hpp:71-75),
measured on the device.  The reference-side comparison (same records as the reference
DpProvider under run_md) is in oracle/provider_md.cpp (tests/test_gpu_integration.py)."""
import json

import numpy as np
import pytest

import paper_2604_07276_b200 as nb

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("scheme", [nb.MASKED_REDUCTION, nb.WIDE_HALO])
def test_spans_and_ledger_of_a_decomposed_step(scheme, tmp_path):
    box, pos, sp = nb.synth_system(600, 0.1, 0.9, 3)
    m = nb.init_model(nb.test_spec(4.0, n_species=6), 1)
    R = 2
    ev = nb.DeviceEvaluator(m, n_ranks=R, scheme=scheme)
    ev.set_trace(True, True)
    for step in range(3):
        ev.set_step(step)
        ev.compute(pos, sp, box)
    spans = ev.trace_spans()
    keys = sorted((r, p, s) for r, p, _, _, s in spans)
    want = []
    for s in range(3):
        want += [(-1, "gather_positions", s), (-1, "reduce_forces", s)]
        if scheme == nb.MASKED_REDUCTION:
            want.append((-1, "ghost_force_route", s))
        for r in range(R):
            want += [(r, "dd_build", s), (r, "neighbor_build", s), (r, "inference", s)]
    assert keys == sorted(want)
    for _, _, t0, t1, _ in spans:
        assert t1 >= t0
    led = ev.ledger()
    n = len(pos)
    routed = sum(ev.rank_stats(r)["route_entries"] for r in range(R))
    for s in range(3):
        recs = [(k, b, p) for st, k, b, p in led if st == s]
        exp = [("gather_positions", 20 * n, R)]
        if scheme == nb.MASKED_REDUCTION:
            exp.append(("ghost_force_route", 20 * routed, R))
        exp.append(("reduce_forces", 12 * n, R))
        assert recs == exp
    path = str(tmp_path / "trace.json")
    ev.export_chrome_trace(path)
    ev_json = json.load(open(path))
    assert len(ev_json) == len(spans)
    assert {e["name"] for e in ev_json} >= {"dd_build", "inference", "gather_positions"}
    assert all(e["ph"] == "X" and e["dur"] >= 0 and "step" in e["args"] for e in ev_json)
    ev.clear_trace()
    assert ev.trace_spans() == [] and ev.ledger() == []


def test_md_loop_records_integrate_spans():
    box, pos, sp = nb.synth_system(300, 0.1, 0.9, 4)
    m = nb.init_model(nb.test_spec(4.0, n_species=6), 1)
    ev = nb.DeviceEvaluator(m, n_ranks=2)
    ev.set_trace(True, True)
    vel = np.zeros_like(pos)
    mass = np.full(len(pos), 12.0)
    ev.run_md(np.ascontiguousarray(pos), vel, mass, sp, box, 0.0005, 4)
    spans = ev.trace_spans()
    integ = sorted(s for r, p, _, _, s in spans if p == "integrate")
    assert integ == [0, 1, 2, 3]
    assert sorted({s for _, _, _, _, s in spans}) == [0, 1, 2, 3]
