"""SSCAPT v1 replay on the device, against dumps the reference wrote.

Rebuild-from-the-dump-alone, as the reference's tests/test_env.py:182-213 and
``stridesim replay`` (cli.py:187-228, bridge.py:325-349) do: the EnvCfg comes
from the dump's config JSON, the field table from its metadata (including the
actuator gain fields, registered before the restore), the heightfield is
regenerated from the config's seed; then ``restore(frame k)`` + one
``StepPipeline.substep`` on the CUDA path must land on frame k+1.

* reference-written dump -> CUDA replay: within 1e-9 (the kernels round every
  + - * / like numpy; only sin/cos may differ from glibc by an ulp), contact
  flags implied by the frames exact;
* CUDA-written dump (a full fused-step run, NaN-triggered) -> rebuilt CUDA
  model replay: bit-exact, every non-boundary frame.
"""

import os

import numpy as np
import pytest

from helpers import GOLDEN

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


def _rebuild(dump):
    """Model, terrain, pipeline and state from a dump alone (tests/test_env.py:192-207)."""
    from paper_2601_22074_b200.capture import restore_model_fields
    from paper_2601_22074_b200.config import EnvCfg, from_dict
    from paper_2601_22074_b200.sim import BatchState, StepPipeline, compile_model
    from paper_2601_22074_b200.terrain import generate_grid

    cfg = from_dict(EnvCfg, dump.config)
    model = compile_model(cfg.scene.model, dump.n_worlds)
    for name, info in dump.metadata["fields"].items():
        if name not in model.field_names():
            model.register_field(name, np.asarray(info["value"], dtype=np.float64))
    restore_model_fields(model, dump.metadata["fields"])
    terrain = generate_grid(cfg.scene.terrain, cfg.seed)
    return StepPipeline(model, terrain), BatchState(model)


def _np(t):
    return t.detach().cpu().numpy()


@pytest.mark.parametrize("name,pairs", [("capture_flat.bin", 15), ("capture_nan.bin", 4)])
def test_replay_reference_dump_on_device(name, pairs):
    from paper_2601_22074_b200.capture import load_capture
    from paper_2601_22074_b200.sim import restore

    d = load_capture(os.path.join(GOLDEN, name))
    pipe, state = _rebuild(d)
    checked = 0
    for k in range(len(d.frames) - 1):
        if k % 4 == 3 or not np.isfinite(d.frames[k + 1].qd).all():
            continue
        restore(state, d.frames[k])
        pipe.substep(state)
        np.testing.assert_allclose(_np(state.q), d.frames[k + 1].q, rtol=1e-9, atol=1e-9, err_msg=f"q frame {k}")
        np.testing.assert_allclose(_np(state.qd), d.frames[k + 1].qd, rtol=1e-9, atol=1e-9, err_msg=f"qd frame {k}")
        checked += 1
    assert checked >= pairs


def test_device_dump_rebuilt_and_replayed_bit_exact(tmp_path):
    """A Velocity-Rough run with the fused step dumps itself on a nonfinite world; a model rebuilt from
    that file alone replays every in-step frame pair bit for bit."""
    from paper_2601_22074_b200.capture import load_capture
    from paper_2601_22074_b200.env import ManagerBasedRlEnv
    from paper_2601_22074_b200.policies import random_policy
    from paper_2601_22074_b200.sim import restore
    from paper_2601_22074_b200.tasks import make_env_cfg

    cfg = make_env_cfg("Velocity-Rough", num_envs=64, seed=9)
    cfg.capture_len = 40
    cfg.capture_dir = str(tmp_path)
    env = ManagerBasedRlEnv(cfg, "Velocity-Rough")
    env.reset()
    for i in range(12):
        env.step(random_policy(env, i, fused=True))
    env.state.qd[5, 0] = float("inf")
    env.step(random_policy(env, 12, fused=True))
    env.synchronize()
    assert len(env.dump_paths) == 1
    d = load_capture(env.dump_paths[0])
    assert d.metadata["nonfinite_worlds"] == [5] and len(d.frames) == 40
    pipe, state = _rebuild(d)
    checked = 0
    for k in range(len(d.frames) - 1):
        if k % 4 == 3 or not np.isfinite(d.frames[k + 1].qd).all():
            continue
        restore(state, d.frames[k])
        pipe.substep(state)
        assert np.array_equal(_np(state.q), d.frames[k + 1].q), f"q frame {k}"
        assert np.array_equal(_np(state.qd), d.frames[k + 1].qd), f"qd frame {k}"
        checked += 1
    assert checked >= 25
