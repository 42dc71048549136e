"""Byte-identical CSV artifacts from the DEVICE replay:
every golden scenario replayed in one batched launch sequence, materialised
by paper_2512_18725_b200.csvio, hashed against the reference's own files
(tests/golden/csv_golden.json); and `csvio.simulate` end to end from a
profile CSV + scenario JSON (the reference CLI's `simulate`, `cli.py:72-125`)."""
import hashlib
import json
import os

import pytest

from tests import _golden

pytestmark = pytest.mark.gpu
GOLD = json.load(open(os.path.join(_golden.HERE, "csv_golden.json")))


def test_device_replay_artifacts_hash_equal_reference():
    from paper_2512_18725_b200 import csvio, engine
    from paper_2512_18725_b200.workload import scenario_from_dict

    names = sorted(GOLD)
    bad = []
    for tname in _golden.table_names():
        group = [n for n in names if str(_golden.replay()[n + "/table"]) == tname]
        tab = _golden.table(tname)
        pipe, h = engine.run_batch([_golden.spec(n) for n in group], tab)
        for i, n in enumerate(group):
            v = pipe.scenario(h, i)
            assert v["status"] == 0, n
            files = csvio.scenario_csvs(scenario_from_dict(_golden.spec(n)), tab, v, segments=True)
            assert sorted(files) == sorted(GOLD[n]), n
            bad += [(n, f) for f, data in files.items() if hashlib.sha256(data).hexdigest() != GOLD[n][f]["sha256"]]
    assert not bad, bad


def test_simulate_writes_reference_files(tmp_path):
    from paper_2512_18725_b200 import csvio
    from paper_2512_18725_b200.profiles import gen_synthetic_profiles, write_profiles
    from paper_2512_18725_b200.workload import save_scenario, scenario_from_dict

    prof = tmp_path / "default.csv"
    write_profiles(gen_synthetic_profiles(), prof)
    scen = tmp_path / "mixed_three_model.json"
    save_scenario(scenario_from_dict(_golden.spec("bundled_seed7")), scen)
    csvio.simulate(prof, [scen], tmp_path / "out", seeds=[0, 7], segments=True, verbose=False)
    for seed in (0, 7):
        got = csvio.sha256_dir(tmp_path / "out" / f"mixed_three_model_seed{seed}")
        assert got == {f: v["sha256"] for f, v in GOLD[f"bundled_seed{seed}"].items()}
    man = json.loads((tmp_path / "out" / "manifest.json").read_text())
    assert man["seeds"] == [0, 7] and man["tool_version"] == "0.1.0" and len(man["config_sha256"]) == 64
