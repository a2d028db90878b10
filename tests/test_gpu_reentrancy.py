"""anneal() is reentrant on distinct problems (reference SPEC.md:240; SURVEY.md
8(b): callable concurrently from distinct host threads, one stream per call):
four Python threads (the binding releases the GIL around device work) anneal
four different graphs at once, exact mode; every result equals its golden
vector (the compiled reference's output) bit for bit."""
import threading

import numpy as np
import pytest

import paper_1908_00210_b200 as pi
from tests.helpers import fnv_rows, golden_configs, product_graph

pytestmark = pytest.mark.gpu


def test_concurrent_anneals_on_distinct_graphs_match_goldens():
    names = ["G1", "G22", "G55", "G81pm1"]
    docs = golden_configs()
    probs = {k: pi.MinCutProblem.with_default_coefficients(product_graph(docs[k]["recipe"])) for k in names}
    results, errors = {}, []
    start = threading.Barrier(len(names) * 2)

    def work(name, run):
        try:
            p = pi.AnnealParams()
            p.sweeps, p.deterministic, p.seed = docs[name]["sweeps"], True, docs[name]["runs"][run]["seed"]
            start.wait()
            results[(name, run)] = pi.anneal(probs[name], p)
        except Exception as e:  # surfaced below
            errors.append((name, run, repr(e)))

    threads = [threading.Thread(target=work, args=(k, r)) for k in names for r in (0, 1)]
    for t in threads:
        t.start()
    for t in threads:
        t.join(timeout=600)
    assert not errors, errors
    for (name, run), res in results.items():
        gold = docs[name]["runs"][run]
        state = np.asarray(res.state, dtype=np.int8).reshape(1, -1)
        assert res.trace[-1].cut == gold["cut"] and res.trace[-1].imbalance == gold["imbalance"], (name, run)
        assert f"{fnv_rows(state)[0]:016x}" == gold["spins_fnv"], (name, run)
    assert len(results) == 8
