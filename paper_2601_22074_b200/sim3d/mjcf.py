"""Subset MJCF loader for the 3-D path: MuJoCo XML -> ModelBuilder -> Model.

mjlab describes robots in MJCF (§3); the reference has no MJCF
support. This loader covers the subset the 3-D kernels simulate:

* ``<option timestep gravity>``; ``<compiler angle="radian|degree">``;
* ``<default>`` classes (nested, ``childclass`` on bodies, ``class`` on
  elements) for ``joint`` / ``geom`` / ``position`` attributes;
* ``<worldbody>`` bodies (``pos``, ``quat``, ``euler`` (xyz), ``axisangle``),
  ``<inertial pos quat mass diaginertia>``, ``<joint type="hinge">`` (``axis``
  ``pos`` ``range`` ``damping`` ``armature``), ``<freejoint/>`` /
  ``type="free"``, ``<geom type="plane|sphere|capsule|box">`` (``size``,
  ``pos``, ``quat``, ``fromto``, ``friction``, ``contype``, ``conaffinity``);
* ``<actuator><position joint kp kv forcerange>``;
* ``<contact><exclude body1 body2/>`` (body pairs that never collide).

Unsupported elements (mesh geoms, sites, sensors, tendons, equality
constraints, explicit contact pairs, geoms with ``condim`` other than 1 / 3,
slide / ball joints, other actuator types) are skipped with a warning, except
joints, which raise (the dynamics would be wrong without them). A terrain is taken from a world plane geom, or added with
``terrain=`` ("plane" or a ModelBuilder.heightfield argument tuple).
"""

from __future__ import annotations

import warnings
import xml.etree.ElementTree as ET

import numpy as np

from .model import (ACT_IMPLICIT, GEOM_BOX, GEOM_CAPSULE, GEOM_PLANE, GEOM_SPHERE, Model, ModelBuilder, ModelError,
                    Opt, axis_angle, quat_mul)

_GEOMS = {"sphere": GEOM_SPHERE, "capsule": GEOM_CAPSULE, "box": GEOM_BOX, "plane": GEOM_PLANE}


def _vec(s, n=None):
    v = np.array([float(x) for x in s.split()], dtype=np.float64)
    if n is not None and v.size != n:
        raise ModelError(f"expected {n} numbers, got {s!r}")
    return v


class _Defaults:
    """Default-class tree: class name -> {element tag: {attr: value}} with inheritance."""

    def __init__(self, root):
        self.classes: dict[str, dict[str, dict[str, str]]] = {"main": {}}
        self.parent: dict[str, str | None] = {"main": None}
        for d in root.findall("default"):
            self._walk(d, None)

    def _walk(self, node, parent):
        name = node.get("class", "main")
        self.parent[name] = parent
        attrs = self.classes.setdefault(name, {})
        for child in node:
            if child.tag == "default":
                self._walk(child, name)
            else:
                attrs.setdefault(child.tag, {}).update(child.attrib)

    def resolve(self, tag, cls):
        chain = []
        c = cls
        while c is not None:
            chain.append(c)
            c = self.parent.get(c)
        if "main" not in chain:
            chain.append("main")
        out: dict[str, str] = {}
        for c in reversed(chain):
            out.update(self.classes.get(c, {}).get(tag, {}))
        return out


def load_mjcf(xml: str, terrain=None, opt: Opt | None = None) -> Model:
    """Compile MJCF text (or a path to an MJCF file) into a Model."""
    text = xml
    if "<mujoco" not in xml:
        with open(xml) as fh:
            text = fh.read()
    root = ET.fromstring(text)
    if root.tag != "mujoco":
        raise ModelError("not an MJCF document (<mujoco> root expected)")
    degree = True
    comp = root.find("compiler")
    if comp is not None and comp.get("angle", "degree") == "radian":
        degree = False
    o = opt or Opt()
    opt_el = root.find("option")
    if opt_el is not None:
        if "timestep" in opt_el.attrib:
            o.timestep = float(opt_el.get("timestep"))
        if "gravity" in opt_el.attrib:
            o.gravity = tuple(_vec(opt_el.get("gravity"), 3))
    defaults = _Defaults(root)
    b = ModelBuilder(root.get("model", "mjcf"), o)
    wb = root.find("worldbody")
    if wb is None:
        raise ModelError("MJCF without <worldbody>")

    def ang(x):
        return np.deg2rad(x) if degree else x

    def frame_quat(el):
        if "quat" in el.attrib:
            q = _vec(el.get("quat"), 4)
            return q / np.linalg.norm(q)
        if "euler" in el.attrib:  # MuJoCo default eulerseq "xyz" (intrinsic)
            e = ang(_vec(el.get("euler"), 3))
            q = np.array([1.0, 0, 0, 0])
            for axis, a in zip(np.eye(3), e):
                q = quat_mul(q, axis_angle(axis, a))
            return q
        if "axisangle" in el.attrib:
            v = _vec(el.get("axisangle"), 4)
            return axis_angle(v[:3], ang(v[3]))
        return np.array([1.0, 0, 0, 0])

    # terrain first (the builder requires it as geom 0)
    plane = [g for g in wb.findall("geom") if defaults.resolve("geom", g.get("class", "main")).get(
        "type", g.get("type", "sphere")) == "plane" or g.get("type") == "plane"]
    if terrain is None or terrain == "plane":
        attrs = dict(defaults.resolve("geom", plane[0].get("class", "main")), **plane[0].attrib) if plane else {}
        b.plane(friction=float(attrs.get("friction", "1").split()[0]))
        b.geoms[0]["contype"] = int(attrs.get("contype", "1"))
        b.geoms[0]["conaffinity"] = int(attrs.get("conaffinity", "1"))
    else:
        b.heightfield(*terrain)

    def add_geom(bid, el, cls):
        a = dict(defaults.resolve("geom", el.get("class", cls)), **el.attrib)
        t = a.get("type", "sphere")
        if t == "plane":
            if bid != 0:
                raise ModelError("planes are only supported on the world body")
            return
        if t not in _GEOMS:
            warnings.warn(f"MJCF geom type {t!r} skipped (unsupported)")
            return
        condim = int(a.get("condim", "3"))
        if condim not in (1, 3):
            warnings.warn(f"MJCF geom condim={condim} simulated as condim 3 (pyramidal, sliding friction only)")
            condim = 3
        size = list(_vec(a.get("size", "0")))
        kw = dict(friction=float(a.get("friction", "1").split()[0]), contype=int(a.get("contype", "1")),
                  conaffinity=int(a.get("conaffinity", "1")), name=a.get("name"), condim=condim)
        if "fromto" in a:
            b.geom(bid, _GEOMS[t], size[:1], fromto=_vec(a["fromto"], 6), **kw)
        else:
            b.geom(bid, _GEOMS[t], size, pos=_vec(a.get("pos", "0 0 0"), 3), quat=frame_quat(el), **kw)

    def walk(el, parent_id, cls):
        for child in el:
            if child.tag == "geom" and parent_id == 0:
                continue  # world geoms: the terrain was handled above
            if child.tag == "body":
                ccls = child.get("childclass", cls)
                inert = child.find("inertial")
                mass, inertia, ipos, iquat = 1e-3, np.array([1e-6] * 3), np.zeros(3), np.array([1.0, 0, 0, 0])
                if inert is not None:
                    mass = float(inert.get("mass", "0"))
                    if "diaginertia" in inert.attrib:
                        inertia = _vec(inert.get("diaginertia"), 3)
                    elif "fullinertia" in inert.attrib:
                        raise ModelError("fullinertia is not supported; use diaginertia + quat")
                    ipos = _vec(inert.get("pos", "0 0 0"), 3)
                    iquat = frame_quat(inert)
                bid = b.body(child.get("name", f"body{len(b.bodies)}"), parent_id,
                             pos=_vec(child.get("pos", "0 0 0"), 3), quat=frame_quat(child), mass=mass,
                             inertia=inertia, ipos=ipos, iquat=iquat)
                for sub in child:
                    if sub.tag == "freejoint":
                        b.free_joint(bid, name=sub.get("name"))
                    elif sub.tag == "joint":
                        a = dict(defaults.resolve("joint", sub.get("class", ccls)), **sub.attrib)
                        jt = a.get("type", "hinge")
                        if jt == "free":
                            b.free_joint(bid, name=a.get("name"))
                            continue
                        if jt != "hinge":
                            raise ModelError(f"joint type {jt!r} is not supported (hinge and free only)")
                        limited = a.get("limited", "auto")
                        rng = None
                        if "range" in a and limited != "false":
                            rng = tuple(ang(_vec(a["range"], 2)))
                        b.hinge(bid, _vec(a.get("axis", "0 0 1"), 3), name=a.get("name"),
                                pos=_vec(a.get("pos", "0 0 0"), 3), range=rng, damping=float(a.get("damping", "0")),
                                armature=float(a.get("armature", "0")))
                    elif sub.tag == "geom":
                        add_geom(bid, sub, ccls)
                    elif sub.tag not in ("body", "inertial"):
                        warnings.warn(f"MJCF element <{sub.tag}> skipped (unsupported)")
                walk(child, bid, ccls)

    walk(wb, 0, "main")
    for tag in ("equality", "tendon", "sensor"):
        sec = root.find(tag)
        if sec is not None and len(sec):
            warnings.warn(f"MJCF <{tag}> section skipped (unsupported): {len(sec)} element(s)")
    con = root.find("contact")
    if con is not None:
        for c_el in con:
            if c_el.tag == "exclude":
                b.exclude_pair(c_el.get("body1"), c_el.get("body2"))
            else:
                warnings.warn(f"MJCF contact <{c_el.tag}> skipped (excludes only)")
    act = root.find("actuator")
    if act is not None:
        for a_el in act:
            if a_el.tag != "position":
                warnings.warn(f"MJCF actuator <{a_el.tag}> skipped (position only)")
                continue
            a = dict(defaults.resolve("position", a_el.get("class", "main")), **a_el.attrib)
            fr = _vec(a["forcerange"], 2) if "forcerange" in a else np.array([-1e9, 1e9])
            b.actuator(a["joint"], kind=ACT_IMPLICIT, kp=float(a.get("kp", "1")), kv=float(a.get("kv", "0")),
                       effort=float(max(abs(fr[0]), abs(fr[1]))))
    return b.compile()
