"""Configuration surface of the B200 env: every dataclass a user of the
reference builds an ``EnvCfg`` from, plus JSON round-trip and hashing.

The field names, defaults and the ``kind`` discriminators follow the
reference so that configs (and capture dumps that embed them) move between
the two implementations unchanged:

* model spec       -- sim/spec.py:27-104
* actuators        -- actuators.py:37-97
* terrain          -- terrain.py:32-103
* manager terms    -- managers/base.py:77-144
* scene / env      -- env.py:55-92, sensors.py:20-23, sensors.py:54-56

Serialization (``to_dict`` / ``from_dict`` / ``config_hash``) reproduces the
reference's canonical JSON (config.py:53-123) byte for byte, because the hash
is embedded in capture dumps and checked on replay.
"""

from __future__ import annotations

import dataclasses
import hashlib
import json
import types
import typing
from dataclasses import dataclass, field
from typing import Any, Union

# ---------------------------------------------------------------------------
# errors


class ConfigError(Exception):
    pass


class SpecError(ValueError):
    """A model description violates a structural constraint (sim/spec.py:23)."""


# ---------------------------------------------------------------------------
# variant registry: dataclasses told apart by their ``kind`` field

_VARIANTS: dict[str, type] = {}


def register_variant(cls: type) -> type:
    kinds = {f.name: f for f in dataclasses.fields(cls)}
    if "kind" not in kinds:
        raise ConfigError(f"{cls.__name__} has no 'kind' field")
    _VARIANTS[kinds["kind"].default] = cls
    return cls


# ---------------------------------------------------------------------------
# model spec (sim/spec.py)

SPEC_VERSION = 1


@dataclass
class JointSpec:
    name: str
    parent: int  # -1 = base, else an earlier joint index
    attach_offset: tuple[float, float] = (0.0, 0.0)
    link_length: float = 0.3
    link_mass: float = 0.5
    rotor_inertia: float = 0.1
    damping: float = 0.1
    pos_limits: tuple[float, float] = (-2.5, 2.5)
    soft_limit_fraction: float = 0.9


@dataclass
class ModelSpec:
    name: str = "robot"
    base_mass: float = 8.0
    base_inertia: float = 0.15
    joints: list[JointSpec] = field(default_factory=list)
    feet: list[int] = field(default_factory=list)
    contact_stiffness: float = 2.0e4
    contact_damping: float = 600.0
    tangential_gain: float = 50.0
    friction: float = 1.0
    gravity: float = 9.81
    physics_dt: float = 0.005
    decimation: int = 4
    spec_version: int = SPEC_VERSION

    @property
    def num_joints(self) -> int:
        return len(self.joints)

    @property
    def nq(self) -> int:
        return 3 + len(self.joints)

    def chain_tips(self) -> list[int]:
        used = {j.parent for j in self.joints}
        return [i for i in range(len(self.joints)) if i not in used]

    def validate(self) -> None:
        """Structural checks with the reference's messages (sim/spec.py:74-104)."""

        def need_positive(v: float, what: str) -> None:
            if not v > 0.0:
                raise SpecError(f"{what} must be strictly positive, got {v}")

        need_positive(self.base_mass, "base_mass")
        need_positive(self.base_inertia, "base_inertia")
        need_positive(self.physics_dt, "physics_dt")
        need_positive(self.contact_stiffness, "contact_stiffness")
        if self.decimation < 1:
            raise SpecError(f"decimation must be >= 1, got {self.decimation}")
        seen: set[str] = set()
        for i, j in enumerate(self.joints):
            where = f"joint {i} ({j.name!r})"
            if j.name in seen:
                raise SpecError(f"duplicate joint name {j.name!r}")
            seen.add(j.name)
            if not -1 <= j.parent < i:
                raise SpecError(f"{where}: parent must be -1 (base) or an earlier joint index")
            need_positive(j.link_length, f"{where}: link_length")
            need_positive(j.link_mass, f"{where}: link_mass")
            need_positive(j.rotor_inertia, f"{where}: rotor_inertia")
            if j.damping < 0.0:
                raise SpecError(f"{where}: damping must be >= 0")
            lo, hi = j.pos_limits
            if not lo < hi:
                raise SpecError(f"{where}: pos_limits must satisfy lo < hi, got ({lo}, {hi})")
            if not 0.0 < j.soft_limit_fraction <= 1.0:
                raise SpecError(f"{where}: soft_limit_fraction must be in (0, 1]")
        tips = set(self.chain_tips())
        for f_idx in self.feet:
            if f_idx not in tips:
                raise SpecError(f"feet: joint index {f_idx} is not a chain tip")


def load_model_spec(path: str) -> ModelSpec:
    """YAML schema v1 (sim/spec.py:107-169). Note the tangential-gain default
    of 400 when the file omits it, which differs from the dataclass default."""
    import yaml

    with open(path, "r") as fh:
        doc = yaml.safe_load(fh)
    if not isinstance(doc, dict):
        raise SpecError(f"model spec file {path!r} is not a mapping")
    if doc.get("spec_version") != SPEC_VERSION:
        raise SpecError(
            f"unsupported spec_version {doc.get('spec_version')!r} (expected {SPEC_VERSION})"
        )
    c = doc.get("contact", {})
    joints = []
    for j in doc.get("joints", []):
        joints.append(
            JointSpec(
                name=j["name"],
                parent=int(j["parent"]),
                attach_offset=tuple(j.get("attach_offset", (0.0, 0.0))),
                link_length=float(j.get("link_length", 0.3)),
                link_mass=float(j.get("link_mass", 0.5)),
                rotor_inertia=float(j.get("rotor_inertia", 0.02)),
                damping=float(j.get("damping", 0.05)),
                pos_limits=tuple(j.get("pos_limits", (-2.5, 2.5))),
                soft_limit_fraction=float(j.get("soft_limit_fraction", 0.9)),
            )
        )
    spec = ModelSpec(
        name=doc.get("name", "robot"),
        base_mass=float(doc.get("base_mass", 8.0)),
        base_inertia=float(doc.get("base_inertia", 0.15)),
        joints=joints,
        feet=[int(i) for i in doc.get("feet", [])],
        contact_stiffness=float(c.get("stiffness", 2.0e4)),
        contact_damping=float(c.get("damping", 600.0)),
        tangential_gain=float(c.get("tangential_gain", 400.0)),
        friction=float(c.get("friction", 1.0)),
        gravity=float(doc.get("gravity", 9.81)),
        physics_dt=float(doc.get("physics_dt", 0.005)),
        decimation=int(doc.get("decimation", 4)),
    )
    spec.validate()
    return spec


def save_model_spec(spec: ModelSpec, path: str) -> None:
    import yaml

    out = {
        "spec_version": spec.spec_version,
        "name": spec.name,
        "base_mass": spec.base_mass,
        "base_inertia": spec.base_inertia,
        "contact": {
            "stiffness": spec.contact_stiffness,
            "damping": spec.contact_damping,
            "tangential_gain": spec.tangential_gain,
            "friction": spec.friction,
        },
        "gravity": spec.gravity,
        "physics_dt": spec.physics_dt,
        "decimation": spec.decimation,
        "joints": [
            dict(
                name=j.name,
                parent=j.parent,
                attach_offset=list(j.attach_offset),
                link_length=j.link_length,
                link_mass=j.link_mass,
                rotor_inertia=j.rotor_inertia,
                damping=j.damping,
                pos_limits=list(j.pos_limits),
                soft_limit_fraction=j.soft_limit_fraction,
            )
            for j in spec.joints
        ],
        "feet": list(spec.feet),
    }
    with open(path, "w") as fh:
        yaml.safe_dump(out, fh, sort_keys=False)


# ---------------------------------------------------------------------------
# actuators (actuators.py:37-97)


@register_variant
@dataclass
class IdealPdCfg:
    kind: str = "ideal_pd"
    joint_patterns: list[str] = field(default_factory=lambda: [".*"])
    kp: float = 40.0
    kd: float = 1.0
    effort_limit: float = 30.0


@register_variant
@dataclass
class DcMotorCfg:
    kind: str = "dc_motor"
    joint_patterns: list[str] = field(default_factory=lambda: [".*"])
    kp: float = 40.0
    kd: float = 1.0
    effort_limit: float = 30.0
    saturation_effort: float = 45.0
    velocity_limit: float = 20.0


@register_variant
@dataclass
class MlpActuatorCfg:
    kind: str = "mlp"
    joint_patterns: list[str] = field(default_factory=lambda: [".*"])
    weights_path: str = ""
    error_history: int = 2
    velocity_history: int = 2
    effort_limit: float = 30.0


@register_variant
@dataclass
class DelayedCfg:
    kind: str = "delayed"
    inner: "ActuatorCfg" = field(default_factory=IdealPdCfg)
    latency_range: tuple[float, float] = (0.0, 0.02)
    resample_on_reset: bool = True
    joint_patterns: list[str] = field(default_factory=list)


ActuatorCfg = IdealPdCfg | DcMotorCfg | MlpActuatorCfg | DelayedCfg


# ---------------------------------------------------------------------------
# terrain (terrain.py:32-103)


@register_variant
@dataclass
class FlatCfg:
    kind: str = "flat"
    proportion: float = 1.0


@register_variant
@dataclass
class PyramidStairsCfg:
    kind: str = "pyramid_stairs"
    step_width: float = 0.4
    step_height_range: tuple[float, float] = (0.05, 0.25)
    proportion: float = 1.0


@register_variant
@dataclass
class RandomGridCfg:
    kind: str = "random_grid"
    cell_width: float = 0.45
    height_range: tuple[float, float] = (0.02, 0.12)
    proportion: float = 1.0


@register_variant
@dataclass
class SlopeCfg:
    kind: str = "slope"
    max_slope: float = 0.4
    proportion: float = 1.0


@register_variant
@dataclass
class UniformNoiseCfg:
    kind: str = "uniform_noise"
    amplitude_range: tuple[float, float] = (0.01, 0.06)
    proportion: float = 1.0


@register_variant
@dataclass
class WaveCfg:
    kind: str = "wave"
    amplitude_range: tuple[float, float] = (0.02, 0.1)
    wavelength: float = 2.0
    proportion: float = 1.0


SubTerrainCfg = FlatCfg | PyramidStairsCfg | RandomGridCfg | SlopeCfg | UniformNoiseCfg | WaveCfg


class TerrainError(ValueError):
    pass


@dataclass
class TerrainGridCfg:
    rows: int = 1
    cols: int = 1
    patch_length: float = 8.0
    spacing: float = 0.05
    mode: str = "curriculum"
    spawn_margin: float = 1.0
    sub_terrains: list[SubTerrainCfg] = field(default_factory=lambda: [FlatCfg()])

    def validate(self) -> None:
        if self.rows < 1 or self.cols < 1:
            raise TerrainError("terrain grid needs rows >= 1 and cols >= 1")
        if not self.sub_terrains:
            raise TerrainError("sub_terrains list is empty")
        if self.mode not in ("curriculum", "random"):
            raise TerrainError(f"unknown terrain mode {self.mode!r}")
        ratio = self.patch_length / self.spacing
        if abs(ratio - round(ratio)) > 1e-9:
            raise TerrainError("patch_length must be a multiple of spacing")


# ---------------------------------------------------------------------------
# manager term configs (managers/base.py:77-144)

MAX_DELAY_STEPS = 64
MAX_HISTORY = 32


def _default_actuators() -> dict:
    return {"main": IdealPdCfg()}


@dataclass
class ActionTermCfg:
    joint_patterns: list[str] = field(default_factory=lambda: [".*"])
    actuators: dict[str, ActuatorCfg] = field(default_factory=_default_actuators)
    scale: float = 0.5
    offset_mode: str = "default"
    clip: tuple[float, float] | None = None


@dataclass
class NoiseCfg:
    kind: str = "none"
    scale: float = 0.0


@dataclass
class ObsTermCfg:
    func: str = ""
    clip: tuple[float, float] | None = None
    scale: float | None = None
    noise: NoiseCfg = field(default_factory=NoiseCfg)
    delay_steps: int = 0
    history: int = 1
    params: dict[str, Any] = field(default_factory=dict)


@dataclass
class ObsGroupCfg:
    terms: dict[str, ObsTermCfg] = field(default_factory=dict)
    enable_noise: bool = True


@dataclass
class RewardTermCfg:
    func: str = ""
    weight: float = 1.0
    params: dict[str, Any] = field(default_factory=dict)


@dataclass
class TerminationTermCfg:
    func: str = ""
    time_out: bool = False
    params: dict[str, Any] = field(default_factory=dict)


@dataclass
class EventTermCfg:
    func: str = ""
    mode: str = "reset"
    interval_range: tuple[float, float] | None = None
    params: dict[str, Any] = field(default_factory=dict)


@dataclass
class CurriculumTermCfg:
    func: str = ""
    params: dict[str, Any] = field(default_factory=dict)


def _default_ranges() -> dict:
    return {"vx": (-1.0, 1.0), "pitch_rate": (0.0, 0.0)}


@dataclass
class CommandCfg:
    ranges: dict[str, tuple[float, float]] = field(default_factory=_default_ranges)
    resample_period: float = 10.0
    cap_scale: float = 2.0


# ---------------------------------------------------------------------------
# sensors + scene + env (sensors.py:20-56, env.py:55-92)


@dataclass
class RayScanCfg:
    offsets: tuple[float, ...] = (-0.4, -0.2, 0.0, 0.2, 0.4)


@dataclass
class ContactSensorCfg:
    history_length: int = 3


@dataclass
class InitStateCfg:
    base_pose: tuple[float, float, float] = (0.0, 0.48, 0.0)
    base_vel: tuple[float, float, float] = (0.0, 0.0, 0.0)
    joint_pos: tuple[float, ...] = ()
    joint_vel: tuple[float, ...] = ()


@dataclass
class SceneCfg:
    model: ModelSpec = field(default_factory=ModelSpec)
    terrain: TerrainGridCfg = field(default_factory=TerrainGridCfg)
    num_envs: int = 16
    world_id_offset: int = 0
    init_state: InitStateCfg = field(default_factory=InitStateCfg)
    ray_scan: RayScanCfg = field(default_factory=RayScanCfg)
    contact_history: int = 3
    spawn_offset: float = 0.5


@dataclass
class EnvCfg:
    scene: SceneCfg = field(default_factory=SceneCfg)
    physics_dt: float | None = None
    decimation: int | None = None
    episode_length_s: float = 20.0
    actions: dict[str, ActionTermCfg] = field(default_factory=dict)
    observations: dict[str, ObsGroupCfg] = field(default_factory=dict)
    rewards: dict[str, RewardTermCfg] = field(default_factory=dict)
    terminations: dict[str, TerminationTermCfg] = field(default_factory=dict)
    events: dict[str, EventTermCfg] = field(default_factory=dict)
    commands: CommandCfg = field(default_factory=CommandCfg)
    curriculum: dict[str, CurriculumTermCfg] = field(default_factory=dict)
    capture_len: int = 200
    capture_dir: str = "captures"
    seed: int = 0


# ---------------------------------------------------------------------------
# canonical JSON (config.py:53-123 of the reference)


def to_dict(obj: Any) -> Any:
    if dataclasses.is_dataclass(obj) and not isinstance(obj, type):
        return {f.name: to_dict(getattr(obj, f.name)) for f in dataclasses.fields(obj)}
    if isinstance(obj, dict):
        return {str(k): to_dict(v) for k, v in obj.items()}
    if isinstance(obj, (list, tuple)):
        return [to_dict(v) for v in obj]
    if obj is None or isinstance(obj, (bool, int, float, str)):
        return obj
    raise ConfigError(f"unserializable config value of type {type(obj).__name__}")


def config_hash(obj: Any) -> str:
    payload = json.dumps(to_dict(obj), separators=(",", ":"))
    return hashlib.sha256(payload.encode("utf-8")).hexdigest()


def _union_args(tp: Any) -> tuple | None:
    origin = typing.get_origin(tp)
    if origin is Union or origin is types.UnionType:
        return typing.get_args(tp)
    return None


def from_dict(tp: Any, data: Any) -> Any:
    """Rebuild a typed config tree from ``to_dict`` output."""
    if isinstance(tp, str):
        tp = globals()[tp]
    args = _union_args(tp)
    if args is not None:
        if data is None and type(None) in args:
            return None
        members = [a for a in args if a is not type(None)]
        if isinstance(data, dict) and "kind" in data and data["kind"] in _VARIANTS:
            return from_dict(_VARIANTS[data["kind"]], data)
        return from_dict(members[0], data)
    if dataclasses.is_dataclass(tp):
        hints = typing.get_type_hints(tp, globalns=globals())
        kwargs = {f.name: from_dict(hints[f.name], data[f.name]) for f in dataclasses.fields(tp) if f.name in data}
        return tp(**kwargs)
    origin = typing.get_origin(tp)
    if origin is dict:
        _, vt = typing.get_args(tp)
        return {k: from_dict(vt, v) for k, v in data.items()}
    if origin is list:
        (et,) = typing.get_args(tp)
        return [from_dict(et, v) for v in data]
    if origin is tuple:
        targs = typing.get_args(tp)
        if len(targs) == 2 and targs[1] is Ellipsis:
            return tuple(from_dict(targs[0], v) for v in data)
        return tuple(from_dict(a, v) for a, v in zip(targs, data))
    if tp is float:
        return float(data)
    return data
