"""Record and estimate files: the reference's text
record and PLRE formats pinned byte-for-byte and message-for-message to files
written by the reference itself (tests/golden/files/, make_golden.py files),
plus the binary record format.  CPU only, except the streaming test class."""

import json
import os
import sys

import numpy as np
import pytest

from conftest import GOLDEN

sys.path.insert(0, GOLDEN)
from perturb import record_perturbations, state_perturbations  # noqa: E402

from paper_1602_08604_b200 import MeasurementRecord, OutcomeRecord  # noqa: E402
from paper_1602_08604_b200 import recordio as io  # noqa: E402

FILES = os.path.join(GOLDEN, "files")
MESSAGES = json.load(open(os.path.join(FILES, "messages.json")))


def _lines(name):
    return open(os.path.join(FILES, name)).read().splitlines()


class TestTextRecord:
    @pytest.mark.parametrize("name", ["record_ghz2.txt", "record_random3.txt"])
    def test_reference_file_round_trip_byte_identical(self, tmp_path, name):
        rec = io.read_record(os.path.join(FILES, name))
        out = tmp_path / "again.txt"
        nbytes = io.write_record(rec, out)
        ref = open(os.path.join(FILES, name), "rb").read()
        assert out.read_bytes() == ref and nbytes == len(ref)

    def test_header_fields(self):
        rec = io.read_record(os.path.join(FILES, "record_ghz2.txt"))
        assert (rec.n, rec.shots, rec.seed, rec.state) == (2, 50, 1602, "ghz")
        assert rec.counts.shape == (9, 4) and (rec.counts.sum(axis=1) == 50).all()

    @pytest.mark.parametrize("case", sorted(k.split(":", 1)[1] for k in MESSAGES if k.startswith("record:")))
    def test_error_messages_match_reference(self, tmp_path, case):
        lines = record_perturbations(_lines("record_ghz2.txt"))[case]
        path = tmp_path / "bad.txt"
        path.write_text("\n".join(lines) + ("\n" if lines else ""))
        with pytest.raises(io.RecordFormatError) as exc:
            io.read_record(path)
        assert str(exc.value) == MESSAGES["record:" + case]

    def test_missing_file_raises_oserror(self, tmp_path):
        with pytest.raises(OSError):
            io.read_record(tmp_path / "nope.txt")

    def test_write_validates(self, tmp_path):
        counts = np.full((9, 4), 12, np.int64)
        with pytest.raises(ValueError, match="sums to 48, expected 50"):
            io.write_record(MeasurementRecord(n=2, shots=50, counts=counts), tmp_path / "x.txt")

    def test_outcome_record_writes_its_histogram(self, tmp_path):
        rng = np.random.default_rng(1)
        o = rng.integers(0, 4, size=(9, 50), dtype=np.uint16)
        io.write_record(OutcomeRecord(n=2, shots=50, outcomes=o), tmp_path / "o.txt")
        back = io.read_record(tmp_path / "o.txt")
        np.testing.assert_array_equal(back.counts, OutcomeRecord(n=2, shots=50, outcomes=o).to_counts().counts)


class TestStateFile:
    def test_reference_file_round_trip_byte_identical(self, tmp_path):
        n, rho = io.read_state(os.path.join(FILES, "state_random3.plre"))
        assert n == 3 and rho.shape == (8, 8) and rho.dtype == np.complex128
        assert abs(np.trace(rho) - 1) < 1e-12 and np.allclose(rho, rho.conj().T)
        out = tmp_path / "s.plre"
        nbytes = io.write_state(out, rho, chunk_rows=3)
        ref = open(os.path.join(FILES, "state_random3.plre"), "rb").read()
        assert out.read_bytes() == ref and nbytes == len(ref)

    @pytest.mark.parametrize("case", sorted(k.split(":", 1)[1] for k in MESSAGES if k.startswith("state:")))
    def test_error_messages_match_reference(self, tmp_path, case):
        blob = open(os.path.join(FILES, "state_random3.plre"), "rb").read()
        path = tmp_path / "state.plre"
        path.write_bytes(state_perturbations(blob)[case])
        with pytest.raises(ValueError) as exc:
            io.read_state(path)
        assert str(exc.value).replace(str(path), "<path>") == MESSAGES["state:" + case]

    def test_rejects_non_square(self, tmp_path):
        with pytest.raises(ValueError, match="square"):
            io.write_state(tmp_path / "x", np.zeros((4, 8), np.complex128))


class TestBinaryRecord:
    @pytest.mark.parametrize("n,shots", [(1, 5), (3, 200), (4, 1000), (5, 70000)])
    def test_counts_round_trip(self, tmp_path, n, shots):
        rng = np.random.default_rng(n)
        counts = rng.multinomial(shots, np.full(1 << n, 1.0 / (1 << n)), size=3**n)
        rec = MeasurementRecord(n=n, shots=shots, counts=counts, seed=7, state="maxmixed")
        path = tmp_path / "r.plrb"
        nbytes = io.write_record_binary(rec, path, chunk_rows=4)
        rf = io.open_record(path)
        assert nbytes == os.path.getsize(path) == 256 + rf.nbytes
        assert (rf.n, rf.shots, rf.seed, rf.state, rf.layout) == (n, shots, 7, "maxmixed", io.LAYOUT_COUNTS)
        from paper_1602_08604_b200 import compact_dtype

        assert rf.data.dtype == np.dtype(compact_dtype(shots))
        np.testing.assert_array_equal(rf.to_record().counts, counts)

    def test_outcomes_round_trip(self, tmp_path):
        rng = np.random.default_rng(3)
        o = rng.integers(0, 8, size=(27, 33), dtype=np.uint16)
        path = tmp_path / "o.plrb"
        io.write_record_binary(OutcomeRecord(n=3, shots=33, outcomes=o), path)
        rf = io.open_record(path)
        assert rf.layout == io.LAYOUT_OUTCOMES and rf.seed is None and rf.state is None
        np.testing.assert_array_equal(rf.to_record().outcomes, o)

    def _good(self, tmp_path):
        counts = np.full((9, 4), 5, np.int64)
        path = tmp_path / "g.plrb"
        io.write_record_binary(MeasurementRecord(n=2, shots=20, counts=counts), path)
        return path, path.read_bytes()

    def test_rejects_bad_magic_truncation_and_size(self, tmp_path):
        path, blob = self._good(tmp_path)
        path.write_bytes(b"XXXX" + blob[4:])
        with pytest.raises(io.RecordFormatError, match="bad magic"):
            io.open_record(path)
        path.write_bytes(blob[:100])
        with pytest.raises(io.RecordFormatError, match="truncated"):
            io.open_record(path)
        path.write_bytes(blob[:-1])
        with pytest.raises(io.RecordFormatError, match="size 291 bytes, expected 292"):
            io.open_record(path)
        path.write_bytes(blob[:4] + (9).to_bytes(4, "little") + blob[8:])
        with pytest.raises(io.RecordFormatError, match="version 9"):
            io.open_record(path)

    def test_row_sums_are_validated_on_read(self, tmp_path):
        path, blob = self._good(tmp_path)
        b = bytearray(blob)
        b[256 + 5 * 4] = 6  # setting 5 (YZ), outcome 0: 6 instead of 5 (uint8 counts)
        path.write_bytes(bytes(b))
        with pytest.raises(ValueError, match=r"setting YZ \(index 5\) sums to 21, expected 20"):
            io.open_record(path).to_record()


@pytest.fixture(scope="module")
def lre():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1602_08604_b200 as lre

    return lre


@pytest.mark.gpu
class TestStreamFromFile:
    @pytest.mark.parametrize("n,shots,kind", [(3, 50, "ghz"), (8, 1000, "w"), (9, 300, "ghz"), (10, 70000, "w")])
    def test_counts_file_equals_in_memory(self, lre, tmp_path, n, shots, kind):
        import torch

        st = lre.StateDescriptor(kind, n)
        rec = lre.sample_counts(st, shots, seed=21)
        path = tmp_path / "r.plrb"
        io.write_record_binary(rec, path)
        a = io.reconstruct_file(path, chunk_bytes=1 << 16, as_tensor=True)
        b = lre.reconstruct(rec, project=False, as_tensor=True)
        assert torch.equal(a.theta, b.theta) and torch.equal(a.mu, b.mu)
        assert a.timings["t_ingest_s"] > 0

    def test_outcome_file_equals_counts(self, lre, tmp_path):
        import torch

        n, shots = 9, 1000
        st = lre.StateDescriptor("w", n)
        path = tmp_path / "o.plrb"
        o = lre.sample_outcomes(st, shots, seed=4)
        io.write_record_binary(o, path)
        a = io.reconstruct_file(path, chunk_bytes=1 << 20, as_tensor=True)
        b = lre.reconstruct(lre.sample_counts(st, shots, seed=4), project=False, as_tensor=True)
        assert torch.equal(a.theta, b.theta)

    def test_bad_row_in_file_raises_reference_message(self, lre, tmp_path):
        n, shots = 4, 100
        rec = lre.sample_counts(lre.StateDescriptor("ghz", n), shots, seed=2).to_host()
        counts = rec.counts.copy()
        path = tmp_path / "r.plrb"
        io.write_record_binary(rec, path)
        blob = bytearray(path.read_bytes())
        blob[256 + 40 * 16] += 1  # setting 40, uint8 counts
        path.write_bytes(bytes(blob))
        from paper_1602_08604_b200 import pauli

        want = f"setting {pauli.setting_label(40, n)} (index 40) sums to {int(counts[40].sum()) + 1}, expected {shots}"
        with pytest.raises(ValueError, match=want.replace("(", r"\(").replace(")", r"\)")):
            io.reconstruct_file(path, chunk_bytes=1 << 10)

    def test_state_file_from_device(self, lre, tmp_path):
        res = lre.reconstruct(lre.sample_counts(lre.StateDescriptor("ghz", 6), 500, seed=1), as_tensor=True)
        io.write_state(tmp_path / "s.plre", res.rho, chunk_rows=7)
        n, rho = io.read_state(tmp_path / "s.plre")
        assert n == 6 and np.array_equal(rho, res.rho.cpu().numpy())
