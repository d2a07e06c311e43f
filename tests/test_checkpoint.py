"""CPU: the checkpoint container (paper_1507_07548_b200/checkpoint.py)
against checkpoints written by the unmodified reference
(tmd::Engine::checkpoint_bytes, src/engine.cpp:420-462; golden vectors from
tests/golden/make_golden.py): parse + re-emit byte for byte, the fresh-engine
metadata layout, and the reference's error messages on truncated data."""
from __future__ import annotations

from pathlib import Path

import numpy as np
import pytest

from host_checkpoint import BlockStat, ByteReader, ByteWriter, EngineCheckpoint
from paper_1507_07548_b200 import IoError

import golden_cases

G = np.load(Path(__file__).resolve().parent / "golden" / "ckpt.npz")


@pytest.mark.parametrize("key", ["sampled_water", "sampled_rf", "fresh_two_clj"])
def test_reference_checkpoints_round_trip(key):
    data = G[key].tobytes()
    c = EngineCheckpoint.from_bytes(data)
    assert c.to_bytes() == data


def test_sampled_checkpoint_contents():
    w = EngineCheckpoint.from_bytes(G["sampled_water"].tobytes())
    comp, _, _ = golden_cases.eval_cases()["water_ions"]
    assert w.config_text == "[system]\nexample = true\n" and w.seed == 7
    assert (w.equil_done, w.prod_done) == (20, 40)
    assert w.state.shape == (comp.molecule_count(), 13) and w.box_length == comp.box_length
    assert w.samplers_ready and w.residence_radius_used > 0.0
    assert w.massieu is None and w.je_corr and w.jq_corr and len(w.vacf) == 3
    assert w.residence and w.rdf and w.rdf_prepass
    rf = EngineCheckpoint.from_bytes(G["sampled_rf"].tobytes())
    assert rf.massieu and rf.jq_corr and rf.je_corr is None and rf.residence is None
    assert all(s.total == 30 for s in rf.stats)


def test_fresh_engine_metadata():
    """A freshly constructed Engine (engine.cpp:63-89) after set_state: seeded
    RNG words, empty single-block statistics, no samplers."""
    data = G["fresh_two_clj"].tobytes()
    meta = EngineCheckpoint.fresh(int(G["fresh_seed"]), n_blocks=10, n_production=0)
    meta.set_state_block(EngineCheckpoint.from_bytes(data).state_block())
    assert meta.to_bytes() == data


@pytest.mark.parametrize("k", range(6))
def test_truncation_messages_match_reference(k):
    data = G["sampled_water"].tobytes()
    cut = int(G["cuts"][k])
    with pytest.raises(IoError) as ei:
        EngineCheckpoint.from_bytes(data[:cut])
    assert str(ei.value) == str(G["cut_messages"][k])


def test_byte_reader_writer_and_block_stat():
    w = ByteWriter()
    w.u8(7), w.u32(9), w.u64(2 ** 40), w.i64(-3), w.f64(1.5), w.str("abc"), w.f64_vec([1.0, 2.0])
    BlockStat(2, 10, 3, [1.0, 2.0], [2, 1]).serialize(w)
    r = ByteReader(w.data())
    assert (r.u8(), r.u32(), r.u64(), r.i64(), r.f64(), r.str(), r.f64_vec()) == \
        (7, 9, 2 ** 40, -3, 1.5, "abc", [1.0, 2.0])
    assert BlockStat.deserialize(r) == BlockStat(2, 10, 3, [1.0, 2.0], [2, 1]) and r.at_end()
    bad = ByteWriter()
    BlockStat(2, 10, 3, [1.0], [1]).serialize(bad)
    with pytest.raises(IoError, match="block stat: corrupted payload"):
        BlockStat.deserialize(ByteReader(bad.data()))
    with pytest.raises(IoError, match="checkpoint: missing end marker"):
        EngineCheckpoint.from_bytes(G["sampled_rf"].tobytes()[:-4] + b"END?")
    with pytest.raises(IoError, match="molecule count mismatch"):
        EngineCheckpoint.from_bytes(G["sampled_rf"].tobytes(), n_molecules=3)
