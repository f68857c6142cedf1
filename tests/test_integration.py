"""The drop-in boundary at the reference's own C++ interface.

integration/locpir/gate_engine.hpp replaces the reference's locpir/gate_engine.hpp
(gate_engine.hpp:1-338) and adds the "tfhe-b200" engine kind over the C ABI.  With it
ahead of the reference's include directory:

* CPU: the reference's UNMODIFIED acceptance test (proj/tests/acceptance.cpp, all eight
  criteria: comparators, the 9-city table through the wire protocol, gate-count model,
  truth tables and refresh noise, determinism) compiles and passes -- the clear and
  tlwe-oracle kinds keep the reference's behaviour through the replacement header.
* GPU: the reference's unmodified loc_pir / hom_less / synthetic_case / zero-sheet
  service flow run on the tfhe-b200 kind (real bootstrapping on the B200): answers equal
  the reference goldens and the counters equal the reference's N(12l+2m+3) model.

Binaries: integration/Makefile (built by __graft_entry__.build() where /root/reference is
present; they travel to the GPU box)."""
import json
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BUILD = os.path.join(ROOT, "integration", "_build")
DRIVER = os.path.join(BUILD, "b200_ref_driver")


def _need(path):
    if not os.path.exists(path):
        pytest.skip(f"{os.path.relpath(path, ROOT)} not built (needs /root/reference at build time)")


def test_reference_acceptance_passes_with_the_replacement_header():
    exe = os.path.join(BUILD, "acceptance_shadow")
    _need(exe)
    if not os.path.isdir("/root/reference/proj/data"):
        pytest.skip("the acceptance test reads the reference's CSV fixture")
    r = subprocess.run([exe], capture_output=True, text=True, timeout=900)
    passes = [ln for ln in r.stdout.splitlines() if ln.startswith("PASS")]
    assert r.returncode == 0 and len(passes) == 8, r.stdout


def _run(*args, timeout=900):
    _need(DRIVER)
    r = subprocess.run([DRIVER, *map(str, args)], capture_output=True, text=True, timeout=timeout)
    line = [ln for ln in r.stdout.splitlines() if ln.startswith("{")][-1]
    d = json.loads(line)
    assert r.returncode == 0 and "error" not in d, (r.stdout, r.stderr[-2000:])
    return d


@pytest.mark.gpu
@pytest.mark.parametrize("sec", [80, 128])
def test_b200_engine_truth_tables(sec):
    d = _run("truth", sec)
    assert d["engine"] == "tfhe-b200"
    want = [0, 0, 0, 1,  0, 1, 1, 1,  0, 1, 1, 0,  1, 0, 0, 1,  1, 0,
            0, 1, 0, 1, 0, 0, 1, 1,  1]
    assert d["bits"] == want and d["refresh"] == 1
    assert d["counters"] == {"and": 5, "or": 4, "xor": 4, "xnor": 4, "not": 2, "mux": 8,
                             "bootstrap_units": 33}


@pytest.mark.gpu
@pytest.mark.parametrize("sec,N,l,m,workers", [(128, 9, 16, 9, 1), (80, 3, 6, 8, 1),
                                               (128, 16, 13, 3, 1), (128, 9, 16, 9, 3),
                                               (80, 1, 32, 16, 2), (128, 20, 13, 16, 1)])
def test_b200_engine_reference_synthetic_case(sec, N, l, m, workers, golden):
    """bench.hpp detail::synthetic_case + circuits.hpp loc_pir, unmodified, on the B200
    engine (workers > 1: the reference's parallel_blocks forks record concurrently)."""
    d = _run("synthetic", sec, N, l, m, workers)
    assert d["got"] == d["expected"] == d["got_sk"]
    assert d["units"] == d["predicted_units"] == N * (12 * l + 2 * m + 3)
    # the reference's own run of the same shape (tests/golden, made by oracle/ref_driver)
    flat = golden["locpir_synthetic_N_l_m_got_expected_units_xnor_mux_and_xor_not_pred"]
    rows = [flat[i:i + 12] for i in range(0, len(flat), 12)]
    for row in rows:
        if row[:3] == [N, l, m]:
            assert d["expected"] == row[4] and d["units"] == row[5]
            c = d["counters"]
            assert [c["xnor"], c["mux"], c["and"], c["xor"], c["not"]] == row[6:11]


@pytest.mark.gpu
@pytest.mark.parametrize("sec", [80, 128])
def test_b200_engine_city_table(sec, golden, tmp_path):
    """The 9-city table (acceptance.cpp:173-237) through the reference's loc_pir with
    zero-sheet services (circuits.hpp:46-146), 9 interior points and one open-sea point."""
    f = tmp_path / "city.txt"
    f.write_text("boxes " + " ".join(map(str, golden["city_boxes_grid_x1_x2_y1_y2_int32"])) + "\n"
                 "services " + " ".join(map(str, golden["city_services"])) + "\n"
                 "bits " + str(golden["city_service_bits"][0]) + "\n"
                 "queries " + " ".join(map(str, golden["city_queries_grid_xy_int32"])) + "\n"
                 "expected " + " ".join(map(str, golden["city_expected"])) + "\n")
    d = _run("city", sec, str(f))
    assert d["got"] == d["expected"] == golden["city_expected"]
    assert d["units"] == len(d["got"]) * d["predicted_units_per_query"]


@pytest.mark.gpu
def test_b200_engine_around_a_reference_key():
    """make_tfhe_b200(SecretKey, ...) around keygen(TlweParams::sec128(), 31): samples the
    reference encrypts with its own NoiseSampler are valid gate inputs."""
    d = _run("refkey")
    assert d["n"] == 630 and d["wrong"] == 0 and d["total"] == 9
