"""Model description types (sim/spec.py of the reference), re-exported."""

from ..config import SPEC_VERSION, JointSpec, ModelSpec, SpecError, load_model_spec, save_model_spec

__all__ = ["SPEC_VERSION", "JointSpec", "ModelSpec", "SpecError", "load_model_spec", "save_model_spec"]
