"""Spill-file format and CLI host logic (CPU, no GPU needed).

The golden spill (tests/golden/ref_spill_small.bin, written by the REAL reference package with
tests/golden/make_spill_golden.py) must read back through this package's reader exactly as the
reference's own open_spill reads it (ref_spill_small.npz), and re-writing its records with this
package's writer must reproduce the file byte for byte (same record framing, payload encoding
and JSON footer: reference cache.py:119-276).
"""

import json

import numpy as np
import pytest


@pytest.fixture(scope="module")
def ref(golden_dir):
    return golden_dir / "ref_spill_small.bin", dict(np.load(golden_dir / "ref_spill_small.npz"))


def test_reads_reference_spill(ref):
    from paper_2305_17423_b200 import spill
    path, want = ref
    foot = spill.read_footer(path)
    assert len(foot["entries"]) == len(want) == 52
    with open(path, "rb") as f:
        for e in foot["entries"]:
            got = spill.decode_payload(spill.read_record(f, e["offset"], e["length"]))
            exp = want[f"{e['step']}_{e['layer']}_{e['role']}"]
            assert got.dtype == np.float32 and got.shape == exp.shape
            assert np.array_equal(got, exp)


def test_rewrite_is_byte_identical(ref, tmp_path):
    from paper_2305_17423_b200 import spill
    path, _ = ref
    foot = spill.read_footer(path)
    out = tmp_path / "re.bin"
    w = spill.SpillWriter(out)
    with open(path, "rb") as f:
        for e in sorted(foot["entries"], key=lambda e: e["offset"]):
            buf = spill.read_record(f, e["offset"], e["length"])
            w.append(e["step"], e["layer"], e["role"], spill.encode_payload(spill.decode_payload(buf)), e["bytes"],
                     e["compacted"])
    w.index.sort(key=lambda r: [x["offset"] for x in foot["entries"]].index(r["offset"]))  # footer order
    w.finish()
    assert out.read_bytes() == path.read_bytes()


def test_compact_payload_roundtrip(tmp_path):
    from paper_2305_17423_b200 import CompactTensor, compact_tensor, spill
    g = np.random.default_rng(3)
    arr = g.standard_normal((1, 5, 8, 8)).astype(np.float32)
    for frac in (0.1, 0.9):
        bits = g.random((8, 8)) < frac
        ct = compact_tensor(arr, bits)
        back = spill.decode_payload(spill.encode_payload(ct))
        assert isinstance(back, CompactTensor) and back.index_is_active == ct.index_is_active
        assert np.array_equal(back.materialize(), ct.materialize())
        assert np.array_equal(back.materialize()[:, :, ~bits], arr[:, :, ~bits])
        assert not back.materialize()[:, :, bits].any()


def test_corrupt_record_and_missing_footer(ref, tmp_path):
    from paper_2305_17423_b200 import ContractViolation, spill
    path, _ = ref
    raw = bytearray(path.read_bytes())
    bad = tmp_path / "bad.bin"
    bad.write_bytes(bytes(raw[:-8]) + b"XXXXXXXX")
    with pytest.raises(ContractViolation):
        spill.read_footer(bad)
    foot = spill.read_footer(path)
    e = foot["entries"][0]
    raw[e["offset"] + 24] ^= 0xFF  # the repeated role byte
    bad.write_bytes(bytes(raw))
    with open(bad, "rb") as f, pytest.raises(ContractViolation):
        spill.read_record(f, e["offset"], e["length"])


def test_cli_usage_errors_and_report_checks(tmp_path):
    from paper_2305_17423_b200 import cli
    assert cli.main([]) == 2
    assert cli.main(["sweep", "--session", str(tmp_path / "nope.json"), "--sizes", "0.1", "--out",
                     str(tmp_path / "s.csv")]) == 2  # missing session -> usage error
    assert cli.main(["sweep", "--session", "x", "--sizes", "1.5", "--out", "y"]) == 2
    (tmp_path / "cfg.json").write_text("{not json")
    assert cli.main(["generate", "--config", str(tmp_path / "cfg.json"), "--prompt", "1", "--out",
                     str(tmp_path / "g")]) == 2
    rec = dict(config_hash="abc", edit_size=0.1, dense_macs=100, sparse_macs=25, macs_ratio=4.0, dense_ms=10.0,
               sparse_ms=2.0, speedup=5.0, cached_bytes_pre=1, cached_bytes_post=1, transfer_bytes=0,
               blocking_loads=0)
    assert cli.BenchReport.from_json({"runs": [rec]}).runs[0].macs_ratio == 4.0
    from paper_2305_17423_b200 import ContractViolation
    with pytest.raises(ContractViolation):
        cli.BenchReport.from_json({"runs": [dict(rec, macs_ratio=3.0)]})
    with pytest.raises(ContractViolation):
        cli.BenchReport.from_json({"runs": [dict(rec, speedup=4.0)]})
    json.dumps(cli.BenchReport.from_json({"runs": [rec]}).to_json())


def test_lcs_pairs_matches_oracle():
    """The package's LCS (SharedTokenMap, reference unet.py:174-195; plain-Python DP rows) returns the
    same pairs as the oracle restatement, ties included, on random and edge-case prompts."""
    import random
    from oracle import sparsedit_oracle as O
    from paper_2305_17423_b200.model import lcs_pairs
    rng = random.Random(7)
    cases = [((), ()), ((1,), ()), ((), (2,)), ((1, 2, 3), (1, 2, 3)), ((1, 2, 3), (3, 2, 1)), ((5, 5, 5), (5, 5))]
    for _ in range(200):
        la, lb = rng.randrange(0, 30), rng.randrange(0, 30)
        cases.append((tuple(rng.randrange(6) for _ in range(la)), tuple(rng.randrange(6) for _ in range(lb))))
    for a, b in cases:
        assert lcs_pairs(a, b) == tuple(O.lcs_pairs(a, b)), (a, b)
