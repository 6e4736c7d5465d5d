"""BenchRecord rows in the reference's pinned CSV schema (SURVEY.md 8f rank
3), so the reference's report tooling (records_from_csv, report.cpp) can read
B200 results next to its own families.

Restates bench.hpp:30-43 (BenchRecord, kCsvHeader) and bench.cpp:38-49
(fmt: shortest round-trip double, sanitize_note), :454-477 (records_to_csv),
:479-525 (records_from_csv).  The run-gpu family's row: experiment
"run-gpu", config_hash = FNV-1a 64 of the canonical workload config (the
reference hashes its INI config, config.cpp, which is out of scope here),
wall_s = device seconds per step, transfer_s = end-to-end host-buffer
seconds per step minus the device part, copy_s = 0, overhead_pct = 0,
imbalance = max/mean per-rank step time - 1 (0 on one GPU), notes =
cols_per_s, roofline_frac, gpus, e2e_cols_per_s, workload, variant.
"""
from __future__ import annotations

import json
import os
from dataclasses import dataclass

CSV_HEADER = "experiment,config_hash,rep,wall_s,overhead_pct,imbalance,copy_s,transfer_s,notes"


@dataclass
class BenchRecord:
    experiment: str
    config_hash: str
    rep: int = 0
    wall_s: float = 0.0
    overhead_pct: float = 0.0
    imbalance: float = 0.0
    copy_s: float = 0.0
    transfer_s: float = 0.0
    notes: str = ""


def fmt(v: float) -> str:
    """std::to_chars shortest round-trip form (bench.cpp:38-42)."""
    v = float(v)
    if v == int(v) and abs(v) < 1e16:
        return str(int(v)) if v != 0 or str(v)[0] != "-" else "-0"
    r = repr(v)
    if "e" in r:
        mant, ex = r.split("e")
        sign = ex[0] if ex[0] in "+-" else "+"
        digits = ex.lstrip("+-").lstrip("0") or "0"
        r = f"{mant}e{sign}{digits.zfill(2)}"
    return r


def sanitize_note(s: str) -> str:
    return s.replace(",", ";").replace("\n", ";").replace("\r", ";")


def records_to_csv(recs) -> str:
    out = [CSV_HEADER]
    for r in recs:
        out.append(",".join([sanitize_note(r.experiment), r.config_hash, str(int(r.rep)), fmt(r.wall_s),
                             fmt(r.overhead_pct), fmt(r.imbalance), fmt(r.copy_s), fmt(r.transfer_s),
                             sanitize_note(r.notes)]))
    return "\n".join(out) + "\n"


def records_from_csv(csv: str):
    lines = csv.splitlines()
    if not lines or lines[0].rstrip("\r") != CSV_HEADER:
        raise ValueError("records: unexpected CSV header")
    recs = []
    for line in lines[1:]:
        line = line.rstrip("\r")
        if not line:
            continue
        parts = line.split(",", 8)
        if len(parts) != 9:
            raise ValueError("records: short row")
        recs.append(BenchRecord(parts[0], parts[1], int(parts[2]), float(parts[3]), float(parts[4]),
                                float(parts[5]), float(parts[6]), float(parts[7]), parts[8]))
    return recs


def config_hash(cfg: dict) -> str:
    """FNV-1a 64 over the canonical JSON of the workload config, 16 hex."""
    h = 0xcbf29ce484222325
    for b in json.dumps(cfg, sort_keys=True, separators=(",", ":")).encode():
        h = ((h ^ b) * 0x100000001b3) & 0xFFFFFFFFFFFFFFFF
    return f"{h:016x}"


def run_gpu_record(line: dict, rep: int = 0) -> BenchRecord:
    """One run-gpu record from a bench.py JSON line."""
    e2e = line.get("e2e") or {}
    dev_s = line["ms_per_step"] * 1e-3
    e2e_s = e2e.get("ms_per_step", 0.0) * 1e-3
    frac = (line.get("step_roofline") or {}).get("frac")
    notes = [f"cols_per_s={fmt(line['value'])}", f"gpus={line['n_gpus']}",
             f"workload={line['config']['workload']}", f"variant={line['config'].get('variant', 0)}"]
    if frac is not None:
        notes.insert(1, f"roofline_frac={fmt(frac)}")
    if e2e:
        notes.append(f"e2e_cols_per_s={fmt(e2e['value'])}")
    par = line.get("parity") or {}
    # flagged_cols: columns exempted from the parity rule;
    # rederived: guard-band levels re-derived exactly; rewritten: count fixes
    notes.append(f"flagged_cols={int(par.get('exempt_columns', 0))}")
    if "rederived_levels" in par:
        notes.append(f"rederived={int(par['rederived_levels'])}")
        notes.append(f"rewritten={int(par['rewritten_patches'])}")
    if "work_mismatch" in par:
        notes.append(f"parity_ok={int(bool(par.get('ok')))}")
    return BenchRecord("run-gpu", config_hash(line["config"]), rep, dev_s, 0.0, line.get("imbalance", 0.0), 0.0,
                       max(e2e_s - dev_s, 0.0) if e2e else 0.0, ";".join(notes))


def append_records(path: str, recs) -> None:
    """Appends rows to a records CSV, writing the header for a new file."""
    new = not os.path.exists(path) or os.path.getsize(path) == 0
    body = records_to_csv(recs)
    with open(path, "a") as f:
        f.write(body if new else body.split("\n", 1)[1])
