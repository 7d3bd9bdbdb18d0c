"""Subset MJCF loader (sim3d/mjcf.py): an MJCF restatement of robots.go1_like, written with default
classes, compiles to the same model arrays as the code-built robot; frame conventions (euler,
axisangle, degrees) and unsupported-element handling."""

import numpy as np
import pytest

from paper_2601_22074_b200.sim3d import robots
from paper_2601_22074_b200.sim3d.mjcf import load_mjcf
from paper_2601_22074_b200.sim3d.model import ModelError

LEGS = (("FR", 1, -1), ("FL", 1, 1), ("RR", -1, -1), ("RL", -1, 1))


def go1_mjcf():
    legs = []
    for leg, sx, sy in LEGS:
        legs.append(f"""
      <body name="{leg}_hip" pos="{0.1881 * sx} {0.04675 * sy} 0">
        <inertial mass="0.68" diaginertia="5e-4 8e-4 6e-4"/>
        <joint name="{leg}_hip_joint" axis="1 0 0" range="-0.86 0.86"/>
        <body name="{leg}_thigh" pos="0 {0.08 * sy} 0">
          <inertial pos="0 0 -0.03" mass="1.0" diaginertia="5e-3 5e-3 1e-3"/>
          <joint name="{leg}_thigh_joint" axis="0 1 0" range="-0.69 4.5"/>
          <geom type="capsule" size="0.02" fromto="0 0 0 0 0 -0.213"/>
          <body name="{leg}_calf" pos="0 0 -0.213">
            <inertial pos="0 0 -0.1" mass="0.2" diaginertia="2e-3 2e-3 1e-4"/>
            <joint name="{leg}_calf_joint" axis="0 1 0" range="-2.82 -0.89"/>
            <geom name="{leg}_foot" type="sphere" size="0.02" pos="0 0 -0.213"/>
          </body>
        </body>
      </body>""")
    acts = "".join(f"""
    <position joint="{leg}_{j}_joint" kp="35" kv="0.5" forcerange="-{e} {e}"/>"""
                   for leg, _, _ in LEGS for j, e in (("hip", 23.7), ("thigh", 23.7), ("calf", 35.55)))
    return f"""<mujoco model="go1_like">
  <compiler angle="radian"/>
  <option timestep="0.005" gravity="0 0 -9.81"/>
  <default>
    <joint armature="0.01"/>
    <geom contype="2" conaffinity="1"/>
  </default>
  <worldbody>
    <geom type="plane" size="0 0 1" contype="1" conaffinity="2"/>
    <body name="trunk" pos="0 0 0.33">
      <freejoint name="trunk_free"/>
      <inertial mass="5.2" diaginertia="0.016 0.037 0.046"/>
      <geom type="box" size="0.19 0.047 0.05"/>{"".join(legs)}
    </body>
  </worldbody>
  <actuator>{acts}
  </actuator>
</mujoco>"""


def test_mjcf_go1_matches_code_built_robot():
    a, b = load_mjcf(go1_mjcf()), robots.go1_like()
    for name in ("body_parentid", "body_pos", "body_quat", "body_mass", "body_inertia", "body_ipos", "jnt_type",
                 "jnt_axis", "jnt_range", "jnt_limited", "dof_armature", "geom_type", "geom_bodyid", "geom_size",
                 "geom_pos", "geom_quat", "geom_contype", "geom_conaffinity", "pair_geom", "actuator_kp",
                 "actuator_kv", "actuator_effort", "qpos0"):
        np.testing.assert_allclose(getattr(a, name), getattr(b, name), atol=1e-12, err_msg=name)
    assert a.jnt_names == b.jnt_names and a.pair_chain == b.pair_chain


def test_mjcf_frames_defaults_and_errors():
    xml = """<mujoco>
  <default>
    <default class="arm"><joint damping="0.5" armature="0.02"/></default>
  </default>
  <worldbody>
    <geom type="plane" size="1 1 1"/>
    <body name="a" pos="0 0 1" euler="90 0 0" childclass="arm">
      <joint name="j1" axis="0 0 1" range="-90 90"/>
      <geom type="sphere" size="0.05"/>
      <body name="b" pos="0.2 0 0" axisangle="0 0 1 90">
        <joint name="j2" axis="0 1 0"/>
        <geom type="mesh" mesh="m"/>
        <site name="s"/>
      </body>
    </body>
  </worldbody>
</mujoco>"""
    with pytest.warns(UserWarning):
        m = load_mjcf(xml)
    np.testing.assert_allclose(m.body_quat[1], [np.cos(np.pi / 4), np.sin(np.pi / 4), 0, 0], atol=1e-12)
    np.testing.assert_allclose(m.body_quat[2], [np.cos(np.pi / 4), 0, 0, np.sin(np.pi / 4)], atol=1e-12)
    np.testing.assert_allclose(m.jnt_range[0], [-np.pi / 2, np.pi / 2], atol=1e-12)  # degrees by default
    assert m.dof_damping.tolist() == [0.5, 0.5] and m.dof_armature.tolist() == [0.02, 0.02]
    assert m.jnt_limited.tolist() == [1, 0]
    with pytest.raises(ModelError):
        load_mjcf(xml.replace('<joint name="j2" axis="0 1 0"/>', '<joint name="j2" type="slide"/>'))


def test_mjcf_contact_excludes_and_skipped_sections():
    """<contact><exclude> removes a body pair's collision candidates (the G1 MJCF's shin / thigh excludes);
    <equality>, <tendon>, <sensor>, explicit <pair>s and condim other than 1 / 3 are reported, not silently
    dropped; condim 1 makes a frictionless pair."""
    base = """<mujoco>
  <worldbody>
    <geom type="plane" size="1 1 1"/>
    <body name="a" pos="0 0 1"><freejoint/><geom type="sphere" size="0.1"/></body>
    <body name="b" pos="0 0 1.15"><freejoint/><geom type="sphere" size="0.1" condim="%s"/></body>
  </worldbody>
  %s
</mujoco>"""
    m = load_mjcf(base % ("3", ""))
    assert [1, 2] in m.pair_geom.tolist()
    m = load_mjcf(base % ("3", '<contact><exclude body1="a" body2="b"/></contact>'))
    assert [1, 2] not in m.pair_geom.tolist() and [0, 1] in m.pair_geom.tolist()
    extra = ('<equality><weld body1="a" body2="b"/></equality><tendon><fixed name="t"/></tendon>'
             '<sensor><accelerometer site="s"/></sensor><contact><pair geom1="x" geom2="y"/></contact>')
    with pytest.warns(UserWarning) as rec:
        load_mjcf(base % ("6", extra))
    msgs = " ".join(str(r.message) for r in rec)
    for word in ("equality", "tendon", "sensor", "pair", "condim=6"):
        assert word in msgs, word
    m = load_mjcf((base % ("1", "")).replace('<geom type="sphere" size="0.1"/>', '<geom type="sphere" size="0.1" condim="1"/>'))
    # a pair takes the larger condim of its geoms (MuJoCo): frictionless between the two spheres only
    assert m.pair_condim[m.pair_geom.tolist().index([1, 2])] == 1 and m.pair_condim[0] == 3
