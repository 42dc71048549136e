"""CSV materialisation: the native repr(float) / csv.writer
formatter (csrc/csv.cu, host code in the C-ABI library) and the artifact
layout of `intfsim simulate` (`cli.py:72-125`), pinned by the SHA-256 of the
reference's own files (tests/golden/csv_golden.json, made by
tests/golden/make_csv_golden.py).  CPU only: replay arrays come from the
oracle; tests/test_gpu_csv.py repeats the hash check on the device replay."""
import csv
import hashlib
import io
import json
import os

import numpy as np
import pytest

import oracle as O
from tests import _golden

GOLD = json.load(open(os.path.join(_golden.HERE, "csv_golden.json")))
EDGE = [0.0, -0.0, 1.0, -1.0, 0.1, 1 / 3, 2 / 3, 1e16, 9999999999999998.0, 1e15, 123456789012345680.0, 1e-4,
        0.0001234, 9.999e-5, 1e-5, 1.5e-5, 5e-324, 2.2250738585072014e-308, 1.7976931348623157e308, 1e22, 1e23,
        1e-7, 123.456, 0.3, 1e100, 1.2345e-100, float("inf"), float("-inf"), 100.0, 1e21, 12345678901234567.0,
        0.5, 2.5e-05, 11.052981161598199]


def test_repr_matches_python_edge_values():
    from paper_2512_18725_b200 import csvio

    for v in EDGE:
        assert csvio.repr_f64(v) == repr(v), v
    assert csvio.repr_f64(float("nan")) == "nan"


def test_repr_matches_python_random():
    from paper_2512_18725_b200 import csvio

    rng = np.random.default_rng(11)
    bits = rng.integers(0, 2**63 - 1, size=40000, dtype=np.int64).view(np.float64)
    vals = np.concatenate([bits[np.isfinite(bits)], rng.uniform(0, 1000, 40000), rng.exponential(5.0, 40000),
                           np.round(rng.uniform(0, 100, 20000), 3), 10.0 ** rng.uniform(-12, 22, 40000)])
    body = csvio.format_rows([(csvio.COL_F64, vals)])
    assert body.decode().split("\r\n")[:-1] == [repr(float(v)) for v in vals]


def test_format_rows_matches_csv_writer():
    from paper_2512_18725_b200 import csvio

    strs = ["plain", "with,comma", 'quo"te', "", "line\nbreak"]
    idx = np.array([0, 1, 2, 3, 4, 0], dtype=np.int32)
    ints = np.array([0, -5, 2**40, 7, 123, 9])
    fl = np.array([0.1, -0.0, 1e16, 3.0, 1e-5, 2 / 3])
    ref = io.StringIO(newline="")
    w = csv.writer(ref)
    w.writerow(["a", "b,c", "d"])
    w.writerows([[int(i), strs[j], repr(float(f)), "np.float64(%r)" % float(f)] for i, j, f in zip(ints, idx, fl)])
    got = csvio.format_rows([(csvio.COL_I64, ints), (csvio.COL_STR, (idx, strs)), (csvio.COL_F64, fl),
                             (csvio.COL_NPF64, fl)], header=["a", "b,c", "d"])
    assert got == ref.getvalue().encode()


def _oracle_files(name):
    from paper_2512_18725_b200 import csvio
    from paper_2512_18725_b200.workload import scenario_from_dict

    d = _golden.spec(name)
    spec = scenario_from_dict(d)
    tab = _golden.table(str(_golden.replay()[name + "/table"]))
    otab = O.TableArrays(tab.models, tab.max_bs, tab.solo, tab.thr)
    rep = O.run_scenario(d, otab)
    assert rep["status"] == 0
    mode = spec.colocation_mode
    X, y, _ = O.samples_from_replay(rep, d, otab, mode.kind == "ewma", float(mode.alpha))
    ids = [m.model_id for m in spec.deployed]
    report = None
    if len(rep["arr_t"]):
        comp = rep["b_completion"][rep["r_batch"]]
        r = O.slo_report([ids[m] for m in rep["arr_model"]], rep["arr_t"], comp, rep["r_slo_met"])
        report = [(m, *vals) for m, vals in r.items()]
    return csvio.scenario_csvs(spec, tab, rep, segments=True, features=(X, y), report=report)


@pytest.mark.parametrize("name", sorted(GOLD))
def test_artifacts_hash_equal_reference_from_oracle_replay(name):
    files = _oracle_files(name)
    assert sorted(files) == sorted(GOLD[name])
    for f, data in files.items():
        assert len(data) == GOLD[name][f]["bytes"], f
        assert hashlib.sha256(data).hexdigest() == GOLD[name][f]["sha256"], f
