"""Freeze the reference's CSV artifacts (SHA-256 + size per file) for every
golden scenario: tests/golden/csv_golden.json.

Runs the UNMODIFIED reference in this container: for each scenario of
make_golden.scenario_list, exactly what `intfsim simulate --segments` writes
(`cli.py:72-125`: arrivals / outcomes / requests / samples / slo_report /
segments through `cli._write_csv`).  The GPU tests re-create the files
through paper_2512_18725_b200.csvio and compare the hashes.

    python tests/golden/make_csv_golden.py
"""
from __future__ import annotations

import hashlib
import json
import os
import sys
import tempfile
from pathlib import Path

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)

import make_golden as mg  # noqa: E402  (puts the reference on sys.path)
from intfsim import colocation, metrics, simcore  # noqa: E402
from intfsim.cli import _write_csv  # noqa: E402
from intfsim.workload import ARRIVAL_CSV_HEADER, arrival_csv_rows, generate_arrivals  # noqa: E402
import intfsim  # noqa: E402


def files_for(spec, table, out: Path) -> dict:
    """The body of `cmd_simulate` for one (scenario, seed) (`cli.py:85-122`)."""
    result = simcore.run_scenario(spec, table)
    _write_csv(out / "arrivals.csv", ARRIVAL_CSV_HEADER, arrival_csv_rows(generate_arrivals(spec)))
    _write_csv(out / "outcomes.csv", simcore.OUTCOME_CSV_HEADER, simcore.outcome_csv_rows(result.outcomes))
    _write_csv(out / "requests.csv", metrics.REQUEST_CSV_HEADER, metrics.request_csv_rows(result.records))
    _write_csv(out / "samples.csv", colocation.SAMPLE_CSV_HEADER,
               colocation.sample_csv_rows(result.samples, spec.colocation_mode))
    if result.records:
        _write_csv(out / "slo_report.csv", metrics.REPORT_CSV_HEADER,
                   metrics.report_csv_rows(metrics.slo_report(result.records)))
    _write_csv(out / "segments.csv", simcore.SEGMENT_CSV_HEADER, simcore.segment_csv_rows(result.outcomes))
    return {p.name: {"sha256": hashlib.sha256(p.read_bytes()).hexdigest(), "bytes": p.stat().st_size}
            for p in sorted(out.glob("*.csv"))}


def main():
    table = intfsim.load_profiles("/root/reference/pkg/profiles/default.csv")
    t16 = mg.table16()
    tabs = {"default": table, "t16": t16[0], "t32": mg.table32()[0]}
    out = {}
    with tempfile.TemporaryDirectory() as tmp:
        for name, spec, tname in mg.scenario_list(table, t16):
            out[name] = files_for(spec, tabs[tname], Path(tmp) / name)
    with open(os.path.join(HERE, "csv_golden.json"), "w") as f:
        json.dump(out, f, indent=1, sort_keys=True)
    print(len(out), "scenarios")


if __name__ == "__main__":
    main()
