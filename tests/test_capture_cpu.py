"""SSCAPT v1 compatibility with the reference, on CPU.

Pinned by dumps the UNMODIFIED reference wrote (tests/golden/make_golden.py
``capture_cases``): ``capture_flat.bin`` is the replay case of the
reference's tests/test_env.py:182-213 (Velocity-Flat, 2 worlds, seed 5, six
zero-action steps, ``env.dump_capture``); ``capture_nan.bin`` is an automatic
nonfinite dump (env.py:240-241, :276-298). Checked here:

* the package's ``load_capture`` parses both field for field, and the dumped
  config rebuilds an ``EnvCfg`` whose ``config_hash`` is the dumped hash;
* the package's writer (``capture.dump_capture``, the one the CUDA env uses)
  re-emits each file BYTE-identically from the parsed frames + metadata;
* replay from the dump alone (model + fields + terrain rebuilt from its
  config/metadata, restore frame k, one substep) reproduces frame k+1 bit for
  bit through the oracle physics (pinned to the reference);
* when /root/reference exists (build container): the reference's own
  ``load_capture`` reads a dump the package wrote from oracle frames, and
  every frame round-trips exactly.
The GPU side (tests/test_gpu_capture.py) replays these dumps on the device.
"""

import json
import os
import sys

import numpy as np
import pytest

from helpers import GOLDEN

REF_SRC = "/root/reference/pkg/src"


class _FrameRing:
    """Duck-typed ring over already-materialized frames (what dump_capture reads)."""

    def __init__(self, dump):
        self._frames = dump.frames
        self.n_worlds, self.nq, self.n_ctrl, self.capacity = dump.n_worlds, dump.nq, dump.n_ctrl, dump.capacity

    def frames(self, pushes=None, count=None):
        return self._frames


@pytest.mark.parametrize("name,n,frames", [("capture_flat.bin", 2, 24), ("capture_nan.bin", 3, 10)])
def test_load_reference_dump(name, n, frames):
    from paper_2601_22074_b200.capture import load_capture
    from paper_2601_22074_b200.config import EnvCfg, config_hash, from_dict

    d = load_capture(os.path.join(GOLDEN, name))
    assert (d.n_worlds, d.nq, d.n_ctrl) == (n, 7, 4)
    assert len(d.frames) == frames
    steps = [f.sim_step for f in d.frames]
    assert steps == list(range(steps[0], steps[0] + frames))
    cfg = from_dict(EnvCfg, d.config)
    assert config_hash(cfg) == d.config_hash
    assert d.task_id in ("Velocity-Flat", "Velocity-Rough")
    assert set(d.metadata) >= {"offending_observation_terms", "offending_reward_terms", "nonfinite_worlds", "fields"}
    for f in d.frames:
        assert f.q.shape == (n, 7) and f.qd.shape == (n, 7) and f.ctrl.shape == (n, 4)


def test_nan_dump_summary_matches_reference_semantics():
    from paper_2601_22074_b200.capture import load_capture

    d = load_capture(os.path.join(GOLDEN, "capture_nan.bin"))
    assert d.metadata["nonfinite_worlds"] == [1]
    hits = d.nonfinite_summary()
    assert any(h["array"] == "qd" and h["world"] == 1 for h in hits)
    assert all(h["world"] == 1 for h in hits)


@pytest.mark.parametrize("name", ["capture_flat.bin", "capture_nan.bin"])
def test_writer_reemits_reference_dump_byte_identical(name, tmp_path):
    from paper_2601_22074_b200.capture import dump_capture, load_capture

    src = os.path.join(GOLDEN, name)
    d = load_capture(src)
    out = str(tmp_path / "again.bin")
    dump_capture(out, _FrameRing(d), d.config_hash, task_id=d.task_id, config_json=d.config, metadata=d.metadata)
    assert open(out, "rb").read() == open(src, "rb").read()


def test_replay_from_reference_dump_bit_exact_on_oracle():
    """tests/test_env.py:182-213 restated: rebuild physics from the dump alone."""
    from oracle.physics import OracleModel, heights_fn, new_state, oracle_substep
    from paper_2601_22074_b200.capture import load_capture
    from paper_2601_22074_b200.config import EnvCfg, from_dict
    from paper_2601_22074_b200.terrain import generate_grid

    d = load_capture(os.path.join(GOLDEN, "capture_flat.bin"))
    cfg = from_dict(EnvCfg, d.config)
    m = OracleModel(cfg.scene.model, d.n_worlds)
    for name, info in d.metadata["fields"].items():
        if name not in m.fields:
            m.add_field(name, np.asarray(info["value"], dtype=np.float64))
        if info.get("expanded"):
            m.expand(name)
        m.fields[name][0][...] = np.asarray(info["value"], dtype=np.float64)
    terrain = generate_grid(cfg.scene.terrain, cfg.seed)
    h = heights_fn(terrain.samples, cfg.scene.terrain.spacing)
    checked = 0
    for k in range(len(d.frames) - 1):
        if k % 4 == 3:  # the next frame follows a control-step boundary (resets / events in between)
            continue
        S = new_state(m)
        S["q"][...] = d.frames[k].q
        S["qd"][...] = d.frames[k].qd
        S["ctrl"][...] = d.frames[k].ctrl
        S["sim_step"] = d.frames[k].sim_step
        oracle_substep(m, h, S)
        assert np.array_equal(S["q"], d.frames[k + 1].q), f"q frame {k}"
        assert np.array_equal(S["qd"], d.frames[k + 1].qd), f"qd frame {k}"
        checked += 1
    assert checked >= 15


@pytest.mark.skipif(not os.path.isdir(REF_SRC), reason="the reference exists only in the build container")
def test_reference_reader_parses_package_dump(tmp_path):
    from oracle import OracleEnv
    from paper_2601_22074_b200.capture import dump_capture
    from paper_2601_22074_b200.config import config_hash, to_dict
    from paper_2601_22074_b200.sim.state import StateFrame
    from paper_2601_22074_b200.tasks import make_env_cfg
    from paper_2601_22074_b200.terrain import generate_grid

    cfg = make_env_cfg("Velocity-Rough", num_envs=5, seed=4)
    cfg.capture_len = 12
    env = OracleEnv(cfg, generate_grid(cfg.scene.terrain, cfg.seed).samples)
    env.reset()
    for _ in range(5):
        env.step(env.random_actions())
    frames = [StateFrame(q, qd, c, s) for q, qd, c, s in env.capture_frames()]

    class Ring:
        n_worlds, nq, n_ctrl, capacity = 5, 7, 4, 12

        def frames(self, pushes=None, count=None):
            return frames

    path = str(tmp_path / "pkg.bin")
    meta = {"offending_observation_terms": [], "offending_reward_terms": [], "nonfinite_worlds": [],
            "fields": {}}
    dump_capture(path, Ring(), config_hash(cfg), task_id="Velocity-Rough", config_json=to_dict(cfg), metadata=meta)
    sys.path.insert(0, REF_SRC)
    try:
        from stridesim.capture import load_capture as ref_load
        from stridesim.config import config_hash as ref_hash
        from stridesim.config import from_dict as ref_from_dict
        from stridesim.env import EnvCfg as RefEnvCfg
    finally:
        sys.path.remove(REF_SRC)
    d = ref_load(path)
    assert (d.n_worlds, d.nq, d.n_ctrl, d.capacity) == (5, 7, 4, 12)
    assert len(d.frames) == len(frames) == 12
    for a, b in zip(frames, d.frames):
        assert np.array_equal(a.q, b.q) and np.array_equal(a.qd, b.qd) and np.array_equal(a.ctrl, b.ctrl)
        assert a.sim_step == b.sim_step
    assert ref_hash(ref_from_dict(RefEnvCfg, d.config)) == d.config_hash == config_hash(cfg)
    assert json.loads(json.dumps(d.metadata)) == meta
