"""Python mirror of the pipetune C++ API (include/pipetune/*.hpp) over the C ABI.

Names follow the reference (proj/include/pipetune/model.hpp:30-51,
plan.hpp:32-49); every call goes through libptk.so — the C++ planner,
simulator and tuner — never through a Python re-implementation.
"""
from __future__ import annotations

import ctypes as C
import json
from dataclasses import dataclass, field

from . import _lib as L

PLAN_1F1B, PLAN_KFKB, PLAN_GPIPE = 0, 1, 2


@dataclass
class StageProfile:
    stage_id: int = 0
    forward_fixed: float = 0.0
    forward_per_sample: float = 0.0
    backward_fixed: float = 0.0
    backward_per_sample: float = 0.0
    weight_bytes: int = 0
    activation_bytes_per_sample: int = 0
    output_bytes_per_sample_fwd: int = 0
    output_bytes_per_sample_bwd: int = 0


@dataclass
class ModelSpec:
    stages: list = field(default_factory=list)
    global_batch: int = 1

    def stage_count(self) -> int:
        return len(self.stages)


class _CStage(C.Structure):
    _fields_ = [
        ("stage_id", C.c_int), ("forward_fixed", C.c_double), ("forward_per_sample", C.c_double),
        ("backward_fixed", C.c_double), ("backward_per_sample", C.c_double), ("weight_bytes", C.c_int64),
        ("activation_bytes_per_sample", C.c_int64), ("output_bytes_per_sample_fwd", C.c_int64),
        ("output_bytes_per_sample_bwd", C.c_int64),
    ]


class _CModel(C.Structure):
    _fields_ = [("stages", C.POINTER(_CStage)), ("stage_count", C.c_int), ("global_batch", C.c_int)]


class PipetuneError(RuntimeError):
    """Carries the C++ exception type name (ConfigError, PlanError, ...)."""

    def __init__(self, kind: str, msg: str = ""):
        super().__init__(f"{kind}: {msg}")
        self.kind = kind


def to_c_model(model: ModelSpec):
    arr = (_CStage * max(1, len(model.stages)))()
    for i, s in enumerate(model.stages):
        for f, _ in _CStage._fields_:
            setattr(arr[i], f, getattr(s, f))
    cm = _CModel(arr, len(model.stages), model.global_batch)
    cm._keep = arr
    return cm


def _call_json(fn, *args) -> dict:
    size = C.c_size_t(0)
    buf = C.create_string_buffer(1 << 16)
    rc = fn(*args, buf, len(buf), C.byref(size))
    if rc == 10:  # PTK_ERR_NOMEM: retry with the size the library asked for
        buf = C.create_string_buffer(size.value)
        rc = fn(*args, buf, len(buf), C.byref(size))
    out = json.loads(buf.value.decode())
    if rc != 0:
        raise PipetuneError(out.get("error", L.STATUS_NAMES.get(rc, str(rc))), L.lib().ptk_last_error().decode())
    return out


def plan_json_str(model: ModelSpec, micro_batch_size: int, kind: int, k: int = 1) -> str:
    lib = L.lib()
    cm = to_c_model(model)
    size = C.c_size_t(0)
    buf = C.create_string_buffer(1 << 16)
    rc = lib.ptk_plan_json(C.byref(cm), micro_batch_size, kind, k, buf, len(buf), C.byref(size))
    if rc == 10:
        buf = C.create_string_buffer(size.value)
        rc = lib.ptk_plan_json(C.byref(cm), micro_batch_size, kind, k, buf, len(buf), C.byref(size))
    return buf.value.decode()


def plan(model: ModelSpec, micro_batch_size: int, kind: int = PLAN_KFKB, k: int = 1) -> dict:
    out = json.loads(plan_json_str(model, micro_batch_size, kind, k))
    if "error" in out:
        raise PipetuneError(out["error"], L.lib().ptk_last_error().decode())
    return out


def plan_kfkb(model: ModelSpec, micro_batch_size: int, k: int) -> dict:
    return plan(model, micro_batch_size, PLAN_KFKB, k)


def plan_1f1b(model: ModelSpec, micro_batch_size: int) -> dict:
    return plan(model, micro_batch_size, PLAN_1F1B)


def plan_gpipe(model: ModelSpec, micro_batch_size: int) -> dict:
    return plan(model, micro_batch_size, PLAN_GPIPE)


def uniform_model(stage_count: int, global_batch: int, fwd_base: int = 10, bwd_base: int = 7,
                  f: float = 1.0, b: float = 2.0) -> ModelSpec:
    """The synthetic model the parity grid uses (mirrors oracle/ref_dump.cpp make())."""
    return ModelSpec([StageProfile(stage_id=s, forward_per_sample=f, backward_per_sample=b,
                                   output_bytes_per_sample_fwd=fwd_base * (s + 1),
                                   output_bytes_per_sample_bwd=bwd_base * (s + 1))
                      for s in range(stage_count)], global_batch)


def scenario(request: dict) -> dict:
    """Run one JSON scenario through the C++ spec modules (ptk_scenario_json)."""
    lib = L.lib()
    req = json.dumps(request).encode()
    size = C.c_size_t(0)
    buf = C.create_string_buffer(1 << 20)
    rc = lib.ptk_scenario_json(req, buf, len(buf), C.byref(size))
    if size.value > len(buf):
        buf = C.create_string_buffer(size.value)
        rc = lib.ptk_scenario_json(req, buf, len(buf), C.byref(size))
    out = json.loads(buf.value.decode())
    if rc != 0:
        raise PipetuneError(out.get("error", str(rc)), out.get("message", ""))
    return out


def model_dict(model: ModelSpec) -> dict:
    return {"global_batch": model.global_batch,
            "stages": [{k: getattr(s, k) for k in StageProfile.__dataclass_fields__} for s in model.stages]}
