"""Bit-exact parity of the exact-mode kernel (K1) with the CPU reference.

Every result here comes from the product path (pyising -> libising -> C ABI
-> sm_100a kernel) and is compared with golden vectors produced by the
unmodified reference (tests/golden, via oracle/_ref) or with the C
restatement (oracle/) on the same seeded inputs. Integer work: bit-exact,
no tolerance.
"""
import numpy as np
import pytest

import paper_1908_00210_b200 as pi
from oracle import oracle as o
from tests.helpers import fnv_rows, golden_configs, product_graph, small_cases

pytestmark = pytest.mark.gpu


@pytest.fixture(autouse=True, params=["auto", "legacy", "exact"])
def kernel_variant(request, monkeypatch):
    """Run every parity test on the exact-mode kernels: k1_block (chosen
    automatically where it fits), k1_window (GDI_FORCE_KERNEL=legacy: the
    automatic choice where k1_block does not fit) and k1_exact."""
    monkeypatch.setenv("GDI_FORCE_KERNEL", request.param)
    return request.param


def det_params(sweeps=1000, pf0=0.04, decay=0.99, seed=1, strategy=pi.Strategy.gdi):
    p = pi.AnnealParams()
    p.sweeps, p.flip_fraction0, p.decay_rate = sweeps, pf0, decay
    p.deterministic, p.seed, p.strategy = True, seed, strategy
    return p


def hexs(xs):
    return [f"{x:016x}" for x in xs]


def check_batch_against_golden(name, count=None, chunk=None):
    doc = golden_configs()[name]
    runs = doc["runs"][:count] if count else doc["runs"]
    g = product_graph(doc["recipe"])
    prob = pi.MinCutProblem.with_default_coefficients(g)
    seeds = np.array([r["seed"] for r in runs], dtype=np.uint64)
    out = pi.anneal_batch(prob, det_params(sweeps=doc["sweeps"]), seeds, trace=True)
    assert out["spins"].shape == (len(runs), doc["n"])
    assert out["cut"].tolist() == [r["cut"] for r in runs]
    assert out["imbalance"].tolist() == [r["imbalance"] for r in runs]
    assert out["hamiltonian_scaled"].tolist() == [r["h_scaled"] for r in runs]
    assert hexs(fnv_rows(out["spins"])) == [r["spins_fnv"] for r in runs]
    assert hexs(fnv_rows(out["trace"].reshape(len(runs), -1))) == [r["trace_fnv"] for r in runs]
    assert out["flip_probability"][-1] == runs[0]["last_pf"]
    head = doc.get("first_full")
    if head and head["seed"] == runs[0]["seed"]:
        assert "".join("1" if v > 0 else "0" for v in out["spins"][0]) == head["spins"]
        assert out["trace"][0].tolist() == head["trace"]
    return out


def test_g1_sixteen_seeds_bit_exact():
    check_batch_against_golden("G1")


def test_g22_1024_replicas_bit_exact():
    out = check_batch_against_golden("G22")
    # trace is internally consistent: last record == final score
    assert (out["trace"][:, -1, 1] == out["cut"]).all()


def test_g55_bit_exact():
    check_batch_against_golden("G55")


def test_g81_pm1_weighted_bit_exact():
    check_batch_against_golden("G81pm1")


@pytest.mark.parametrize("name,best", [("G47", 3364), ("G43", 3374), ("G32", 44)])
def test_acceptance_quality_known_answers(name, best):
    out = check_batch_against_golden(name)
    bal = out["imbalance"] == 0
    assert int(out["cut"][bal].min()) == best


@pytest.mark.parametrize("case", small_cases(), ids=lambda c: c["name"])
def test_small_cases_single_anneal(case):
    g = pi.Graph.from_edges(case["n"], [tuple(e) for e in case["edges"]])
    prob = pi.MinCutProblem.make_unchecked(g, pi.Coefficients(*case["coeffs"]))
    strat = pi.Strategy.standard if case["strategy"] == "standard" else pi.Strategy.gdi
    r = pi.anneal(prob, det_params(case["sweeps"], case["pf0"], case["decay"], case["seed"], strat))
    assert list(r.state) == case["spins"]
    assert [[t.hamiltonian_scaled, t.cut, t.imbalance] for t in r.trace] == case["trace"]
    assert [t.flip_probability for t in r.trace] == case["pf"]
    sc = pi.score(prob, r.state)
    assert (sc.cut, sc.imbalance, sc.hamiltonian_scaled) == (case["cut"], case["imbalance"], case["h_scaled"])


def test_small_cases_batched_seeds_match_oracle():
    # many seeds per small weighted graph in one launch vs the C restatement
    for case in small_cases()[4:12]:
        e = np.array(case["edges"], dtype=np.int64).reshape(-1, 3)
        og = o.csr_from_edges(case["n"], e[:, 0], e[:, 1], e[:, 2])
        g = pi.Graph.from_edges(case["n"], [tuple(x) for x in case["edges"]])
        a, b, d = case["coeffs"]
        prob = pi.MinCutProblem.make_unchecked(g, pi.Coefficients(a, b, d))
        seeds = np.arange(100, 164, dtype=np.uint64)
        out = pi.anneal_batch(prob, det_params(case["sweeps"], case["pf0"], case["decay"]), seeds, trace=True)
        for i, s in enumerate(seeds.tolist()):
            ref = o.anneal(og, s, case["sweeps"], case["pf0"], case["decay"], a, b, d)
            assert out["spins"][i].tolist() == ref["spins"].tolist()
            assert out["trace"][i].tolist() == ref["trace"].tolist()


def test_wide_field_path_matches_oracle():
    # |sum_j w_ij| beyond int32 exercises the 64-bit field variant
    rng = np.random.default_rng(7)
    n, edges, seen = 40, [], set()
    while len(edges) < 120:
        u, v = sorted(rng.integers(0, n, 2).tolist())
        if u == v or (u, v) in seen:
            continue
        seen.add((u, v))
        edges.append((u, v, int(rng.choice([-1, 1])) * int(rng.integers(1 << 28, 1 << 30))))
    e = np.array(edges, dtype=np.int64)
    og = o.csr_from_edges(n, e[:, 0], e[:, 1], e[:, 2])
    prob = pi.MinCutProblem.make_unchecked(pi.Graph.from_edges(n, edges), pi.Coefficients(3, 2, 1))
    seeds = np.arange(1, 33, dtype=np.uint64)
    out = pi.anneal_batch(prob, det_params(50, 0.2, 0.9), seeds, trace=True)
    for i, s in enumerate(seeds.tolist()):
        ref = o.anneal(og, s, 50, 0.2, 0.9, 3, 2, 1)
        assert out["spins"][i].tolist() == ref["spins"].tolist()
        assert out["trace"][i].tolist() == ref["trace"].tolist()


def test_odd_replica_counts_and_reproducibility():
    g = pi.random_graph(300, 1500, 5)
    prob = pi.MinCutProblem.with_default_coefficients(g)
    og = o.random_graph(300, 1500, 5)
    for R in (1, 3, 33, 129):
        seeds = np.arange(7, 7 + R, dtype=np.uint64)
        a = pi.anneal_batch(prob, det_params(40), seeds)
        b = pi.anneal_batch(prob, det_params(40), seeds)
        assert np.array_equal(a["spins"], b["spins"])
        ref = o.anneal(og, 7 + R - 1, 40)
        assert a["spins"][-1].tolist() == ref["spins"].tolist()


def test_evaluate_batch_k3_matches_oracle():
    for recipe in (["random", "2000", "19990", "22"], ["torus_pm1", "100", "200", "81"]):
        g = product_graph(recipe)
        og = o.recipe(":".join(recipe))
        prob = pi.MinCutProblem.with_default_coefficients(g)
        rng = np.random.default_rng(3)
        spins = np.where(rng.random((17, g.num_nodes)) < 0.5, 1, -1).astype(np.int8)
        sc = pi.evaluate_batch(prob, spins)
        for r in range(17):
            cut = o.cut(og, spins[r])
            bal = int(spins[r].astype(np.int64).sum())
            assert sc["cut"][r] == cut
            assert sc["imbalance"][r] == abs(bal)
            assert sc["hamiltonian_scaled"][r] == bal * bal + 4 * cut


def test_session_device_resident_matches_batch(kernel_variant):
    g = pi.random_graph(2000, 19990, 22)
    prob = pi.MinCutProblem.with_default_coefficients(g)
    seeds = np.arange(1, 65, dtype=np.uint64)
    s = pi.Session(prob, det_params(100), 64, trace=True)
    s.set_seeds(seeds)
    s.launch()
    s.sync()
    got = s.fetch(spins=True, trace=True)
    ref = pi.anneal_batch(prob, det_params(100), seeds, trace=True)
    assert np.array_equal(got["spins"], ref["spins"])
    assert np.array_equal(got["trace"], ref["trace"])
    assert s.launch_count >= 1 and s.kernel
    assert ("block" in s.kernel) == (kernel_variant == "auto")
    assert ("window" in s.kernel) == (kernel_variant == "legacy")


def test_window_edge_cases_match_oracle():
    # n just above 2L, dense rows (window masks heavily populated), +-1 weights
    rng = np.random.default_rng(11)
    for n, m, signed in ((64, 300, False), (65, 2000, True), (97, 4000, False), (130, 260, True)):
        seen, edges = set(), []
        while len(edges) < m:
            u, v = sorted(int(x) for x in rng.integers(0, n, 2))
            if u == v or (u, v) in seen:
                continue
            seen.add((u, v))
            edges.append((u, v, int(rng.choice([-1, 1])) if signed else 1))
        e = np.array(edges, dtype=np.int64)
        og = o.csr_from_edges(n, e[:, 0], e[:, 1], e[:, 2])
        prob = pi.MinCutProblem.with_default_coefficients(pi.Graph.from_edges(n, edges))
        seeds = np.arange(1, 41, dtype=np.uint64)
        out = pi.anneal_batch(prob, det_params(30, 0.3, 0.9), seeds, trace=True)
        for i, s in enumerate(seeds.tolist()):
            ref = o.anneal(og, s, 30, 0.3, 0.9)
            assert out["spins"][i].tolist() == ref["spins"].tolist(), (n, m, s)
            assert out["trace"][i].tolist() == ref["trace"].tolist(), (n, m, s)


# ---- global-memory spins (k1_window<...,gmem>): graphs whose spins do not
# fit in shared memory, e.g. the 1M-vertex config (BASELINE configs[4])


@pytest.mark.parametrize("variant", ["window_gmem", "window_masks"])
@pytest.mark.parametrize("name,count", [("G1", 16), ("G22", 256), ("G81pm1", 16)])
def test_forced_exact_variants_bit_exact(name, count, variant, kernel_variant, monkeypatch):
    """The other exact-kernel forms on the golden configs: k1_window with
    global-memory spins and with row-gathered fields (masks)."""
    if kernel_variant != "auto":
        pytest.skip("one forced variant per case")
    monkeypatch.setenv("GDI_FORCE_KERNEL", variant)
    s = pi.Session(pi.MinCutProblem.with_default_coefficients(product_graph(golden_configs()[name]["recipe"])),
                   det_params(), 1)
    assert ("gmem" in s.kernel) == variant.endswith("gmem"), s.kernel
    assert "incf" not in s.kernel, s.kernel
    assert s.kernel.startswith("k1_" + variant.split("_")[0]), s.kernel
    check_batch_against_golden(name, count=count)


def test_m1_million_vertices_bit_exact(kernel_variant):
    if kernel_variant == "exact":
        pytest.skip("k1_exact keeps spins in shared memory: 1M does not fit (capacity)")
    out = check_batch_against_golden("M1")
    assert out["cut"][0] == 1252631 and out["imbalance"][0] == 0


@pytest.mark.parametrize("jt2", ["0", "1"])
def test_window_jump_forms_bit_exact(jt2, kernel_variant, monkeypatch):
    """k1_window's producer jump as the plain bit matrix (configs whose shared
    memory is full) and as the two-column table: same draws, same anneal."""
    if kernel_variant != "legacy":
        pytest.skip("k1_window only")
    monkeypatch.setenv("GDI_WINDOW_JT2", jt2)
    check_batch_against_golden("G22", count=64)


@pytest.mark.parametrize("big", [600, 1800])
def test_exact_results_independent_of_batch_size(big, kernel_variant):
    """Exact mode: a replica's anneal depends on its seed only. Large batches
    change the kernel's shape (replicas per CTA 5 and 13 -> 12, producer lanes
    per stream 4 and 2, more CTAs than SMs at 1800) but not a single spin."""
    if kernel_variant == "exact":
        pytest.skip("k1_block and k1_window only")
    g = product_graph(golden_configs()["G1"]["recipe"])
    prob = pi.MinCutProblem.with_default_coefficients(g)
    p = det_params(sweeps=200)
    small = pi.anneal_batch(prob, p, np.arange(1, 65, dtype=np.uint64), True)
    large = pi.anneal_batch(prob, p, np.arange(1, big + 1, dtype=np.uint64), True)
    assert np.array_equal(small["spins"], large["spins"][:64])
    assert np.array_equal(small["trace"], large["trace"][:64])
