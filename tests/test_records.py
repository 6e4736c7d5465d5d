"""BenchRecord CSV: run-gpu rows in the reference's
pinned schema, parsed and re-serialised by the reference's own
records_from_csv / records_to_csv (bench.cpp:454-525, oracle/_ref)."""
import pytest

import oracle as O
from paper_1711_00289_b200 import records as R

LINE = {"metric": "convective columns/sec (deep+shallow, fp64)", "value": 1396710667.9384682, "n_gpus": 1,
        "ms_per_step": 0.6334425735473633, "config": {"workload": "c4", "n_columns": 884736, "levels": 30,
                                                       "variant": 0},
        "step_roofline": {"frac": 0.44844353932638426},
        "e2e": {"value": 47987623.5, "ms_per_step": 18.43675380005152},
        "parity": {"ok": True, "exempt_columns": 0, "work_mismatch": 0, "rederived_levels": 12509,
                   "rewritten_patches": 77}}


def test_header_is_the_reference_schema():
    if not O.ref_available():
        pytest.skip("reference build missing")
    st, n, text = O.ref_records_roundtrip(R.CSV_HEADER + "\n")
    assert st == 0 and n == 0 and text.splitlines()[0] == R.CSV_HEADER


@pytest.mark.parametrize("v", [0.0, 1.0, 2.5, 1e-05, 0.6334425735473633, 1396710667.9384682, 1e16, 3e-300])
def test_fmt_matches_to_chars(v):
    if not O.ref_available():
        pytest.skip("reference build missing")
    rec = R.BenchRecord("x", "h", 0, v)
    st, n, text = O.ref_records_roundtrip(R.records_to_csv([rec]))
    assert st == 0 and n == 1
    assert text == R.records_to_csv([rec])


def test_run_gpu_record_roundtrips_through_the_reference():
    rec = R.run_gpu_record(LINE)
    csv = R.records_to_csv([rec, R.run_gpu_record(LINE, rep=1)])
    back = R.records_from_csv(csv)
    assert back[0].experiment == "run-gpu" and back[1].rep == 1
    assert "cols_per_s=" in back[0].notes and "roofline_frac=" in back[0].notes and "," not in back[0].notes
    assert "flagged_cols=0" in back[0].notes and "rederived=12509" in back[0].notes and "parity_ok=1" in back[0].notes
    assert abs(back[0].wall_s - LINE["ms_per_step"] * 1e-3) < 1e-15
    if O.ref_available():
        st, n, text = O.ref_records_roundtrip(csv)
        assert st == 0 and n == 2 and text == csv


def test_append_records(tmp_path):
    p = tmp_path / "recs.csv"
    R.append_records(str(p), [R.run_gpu_record(LINE)])
    R.append_records(str(p), [R.run_gpu_record(LINE, rep=1)])
    recs = R.records_from_csv(p.read_text())
    assert [r.rep for r in recs] == [0, 1]
