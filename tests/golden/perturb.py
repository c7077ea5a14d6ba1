"""File perturbations shared by make_golden.py (run against the reference's
readers) and tests/test_recordio.py (run against ours)."""

import json


def record_perturbations(lines):
    """Named perturbations of a good pauli-lre/1 file (mirrors test_records.py:78-140)."""
    out = {}
    L = list(lines)
    label, payload = L[4].split(" ")
    L[4] = label + " " + ",".join(payload.split(",")[:-1])
    out["short_count_line"] = L
    out["body_length"] = list(lines[:-1])
    L = list(lines)
    L[1], L[2] = L[2], L[1]
    out["out_of_order"] = L
    L = list(lines)
    label, payload = L[7].split(" ")
    c = [int(t) for t in payload.split(",")]
    c[0] += 2
    L[7] = label + " " + ",".join(map(str, c))
    out["wrong_sum"] = L
    out["bad_header"] = ["{not json"] + list(lines[1:])
    h = json.loads(lines[0])
    h["format"] = "pauli-lre/9"
    out["format_tag"] = [json.dumps(h)] + list(lines[1:])
    L = list(lines)
    label, payload = L[2].split(" ")
    parts = payload.split(",")
    parts[1] = str(int(parts[1]) + int(parts[0]) + 1)
    parts[0] = "-1"
    L[2] = label + " " + ",".join(parts)
    out["negative"] = L
    L = list(lines)
    L[3] = L[3].split(" ")[0] + " 1.5," + ",".join(L[3].split(" ")[1].split(",")[1:])
    out["non_integer"] = L
    h = json.loads(lines[0])
    h["n"] = 3
    out["header_n"] = [json.dumps(h)] + list(lines[1:])
    h = json.loads(lines[0])
    h["shots"] = "50"
    out["shots_type"] = [json.dumps(h)] + list(lines[1:])
    L = list(lines)
    L[5] = L[5].replace(" ", "")
    out["no_separator"] = L
    out["empty"] = []
    return out


def state_perturbations(blob):
    """Named perturbations of a good PLRE v1 file."""
    return {"truncated": blob[:7], "bad_magic": b"XLRE" + blob[4:],
            "version": blob[:4] + (2).to_bytes(4, "little") + blob[8:], "size": blob[:-16]}
