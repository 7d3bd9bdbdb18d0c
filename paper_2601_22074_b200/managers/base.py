"""Term registries shared by the managers (managers/base.py:1-70).

A term is a registered function plus a typed config. Built-in terms (mdp.py)
carry a ``ss_id`` attribute: the manager lowers them to the fused kernel's
term table and never calls them on the hot path. Any other registered
function is a user plugin: the env evaluates it in Python between kernel
stages (on the device tensors the env exposes) and feeds its values to the
kernel, preserving the reference's stage order.
"""

from __future__ import annotations

from typing import Callable

from ..config import (
    MAX_DELAY_STEPS,
    MAX_HISTORY,
    ActionTermCfg,
    CommandCfg,
    CurriculumTermCfg,
    EventTermCfg,
    NoiseCfg,
    ObsGroupCfg,
    ObsTermCfg,
    RewardTermCfg,
    TerminationTermCfg,
)

__all__ = [
    "MAX_DELAY_STEPS",
    "MAX_HISTORY",
    "ActionTermCfg",
    "CommandCfg",
    "CurriculumTermCfg",
    "EventTermCfg",
    "ManagerError",
    "NoiseCfg",
    "ObsGroupCfg",
    "ObsTermCfg",
    "RewardTermCfg",
    "TerminationTermCfg",
    "OBSERVATION_TERMS",
    "REWARD_TERMS",
    "TERMINATION_TERMS",
    "EVENT_TERMS",
    "CURRICULUM_TERMS",
    "observation_term",
    "reward_term",
    "termination_term",
    "event_term",
    "curriculum_term",
    "resolve",
    "builtin_id",
]


class ManagerError(ValueError):
    pass


OBSERVATION_TERMS: dict[str, Callable] = {}
REWARD_TERMS: dict[str, Callable] = {}
TERMINATION_TERMS: dict[str, Callable] = {}
EVENT_TERMS: dict[str, Callable] = {}
CURRICULUM_TERMS: dict[str, Callable] = {}


def _register(registry: dict, name: str):
    def deco(fn: Callable) -> Callable:
        registry[name] = fn
        return fn

    return deco


def observation_term(name: str):
    return _register(OBSERVATION_TERMS, name)


def reward_term(name: str):
    return _register(REWARD_TERMS, name)


def termination_term(name: str):
    return _register(TERMINATION_TERMS, name)


def event_term(name: str):
    return _register(EVENT_TERMS, name)


def curriculum_term(name: str):
    return _register(CURRICULUM_TERMS, name)


def resolve(registry: dict, func_id: str, what: str) -> Callable:
    if func_id not in registry:
        raise ManagerError(
            f"unknown {what} term function {func_id!r}; registered: {', '.join(sorted(registry)) or 'none'}"
        )
    return registry[func_id]


def builtin_id(fn: Callable) -> int | None:
    """Kernel term id of a built-in term function, None for user plugins."""
    return getattr(fn, "ss_id", None)


def builtin(ss_id: int):
    """Mark a registered function as lowered to kernel term ``ss_id``."""

    def deco(fn: Callable) -> Callable:
        fn.ss_id = ss_id
        return fn

    return deco
