"""Architecture descriptions, launch records and feature vectors.

Mirrors the reference's configuration surface: ``load_arch`` (ls/cost.py:81-129)
with the three builtin targets (ls/archs/*.toml), ``CacheSpec``
(ls/cache.py:19-25), ``SchedSpec`` (ls/ilp.py:18-35), ``GpuSpec`` /
``KernelLaunch`` (ls/ptx.py:15-60) and ``FeatureVector`` (ls/cost.py:33-55).
These are host-side, per-task data; the packer folds them into the task
descriptor (pack.py).
"""

from __future__ import annotations

import math
import tomllib
from dataclasses import dataclass, field
from pathlib import Path

CPU_FEATURES = ("n_fma", "n_vload", "n_vstore", "est_l1_movement", "ilp_cycles")
GPU_FEATURES = ("workload_per_thread", "sm_underuse", "warp_slack",
                "n_smem_ops_adjusted", "n_fma", "n_ld", "n_st")


class CostModelError(ValueError):
    pass


@dataclass(frozen=True)
class FeatureVector:
    values: tuple

    @staticmethod
    def of(mapping: dict, order: tuple) -> "FeatureVector":
        missing = [k for k in order if k not in mapping]
        if missing:
            raise CostModelError(f"missing features: {missing}")
        vals = tuple((k, float(mapping[k])) for k in order)
        for k, v in vals:
            if not (v >= 0.0 and math.isfinite(v)):
                raise CostModelError(f"feature {k} must be finite and >= 0, got {v}")
        return FeatureVector(vals)

    def as_dict(self) -> dict:
        return dict(self.values)

    def __getitem__(self, key: str) -> float:
        for k, v in self.values:
            if k == key:
                return v
        raise KeyError(key)


@dataclass(frozen=True)
class CacheSpec:
    capacity_elements: int

    def __post_init__(self):
        if self.capacity_elements <= 0:
            raise ValueError("cache capacity must be positive")


@dataclass(frozen=True)
class SchedSpec:
    issue_width: int = 4
    latency: dict = None
    default_latency: int = 1
    units: dict = None

    def __post_init__(self):
        if self.issue_width < 1:
            raise ValueError("issue width must be >= 1")
        object.__setattr__(self, "latency", dict(self.latency or {}))
        object.__setattr__(self, "units", dict(self.units or {}))
        if any(v < 1 for v in self.latency.values()):
            raise ValueError("latencies must be >= 1")


DEFAULT_PTX_COSTS = {"fma": 4, "mad": 4, "mul": 4, "add": 2, "sub": 2, "ld": 8, "st": 8,
                     "mov": 1, "setp": 2, "bra": 2, "ret": 1, "bar": 2}


@dataclass(frozen=True)
class GpuSpec:
    num_sms: int = 80
    max_threads_per_sm: int = 2048
    registers_per_sm: int = 65536
    shared_mem_per_sm_bytes: int = 98304
    warp_size: int = 32
    banks: int = 32
    instr_cost: dict = None

    def __post_init__(self):
        object.__setattr__(self, "instr_cost", dict(self.instr_cost or DEFAULT_PTX_COSTS))
        for name in ("num_sms", "max_threads_per_sm", "registers_per_sm", "shared_mem_per_sm_bytes"):
            if getattr(self, name) <= 0:
                raise ValueError(f"{name} must be positive")


@dataclass(frozen=True)
class KernelLaunch:
    grid_blocks: int
    threads_per_block: int
    registers_per_thread: int
    shared_mem_per_block_bytes: int

    def __post_init__(self):
        for name in ("grid_blocks", "threads_per_block", "registers_per_thread"):
            if getattr(self, name) <= 0:
                raise ValueError(f"{name} must be positive")
        if self.shared_mem_per_block_bytes < 0:
            raise ValueError("shared_mem_per_block_bytes must be >= 0")

    @staticmethod
    def from_json(data: dict) -> "KernelLaunch":
        smem = data.get("shared_mem_per_block", data.get("shared_mem_per_block_bytes", 0))
        return KernelLaunch(int(data["grid_blocks"]), int(data["threads_per_block"]),
                            int(data["registers_per_thread"]), int(smem))


def sm_underuse(launch, gpu) -> float:
    """ls/ptx.py:238-241."""
    return max(0, gpu.num_sms - launch.grid_blocks) / gpu.num_sms


def blocks_per_sm(launch, gpu) -> int:
    """ls/ptx.py:244-250."""
    rpb = launch.registers_per_thread * launch.threads_per_block
    limits = (gpu.registers_per_sm // rpb if rpb else gpu.max_threads_per_sm,
              gpu.shared_mem_per_sm_bytes // launch.shared_mem_per_block_bytes
              if launch.shared_mem_per_block_bytes else gpu.max_threads_per_sm,
              gpu.max_threads_per_sm // launch.threads_per_block)
    return max(0, min(limits))


def warp_slack(launch, gpu) -> float:
    """ls/ptx.py:253-256."""
    warps = blocks_per_sm(launch, gpu) * launch.threads_per_block / gpu.warp_size
    return 1.0 / max(1.0, warps)


@dataclass(frozen=True)
class ArchSpec:
    name: str
    family: str
    target: str
    dialect: str
    coefficients: dict
    cache: "CacheSpec | None" = None
    sched: "SchedSpec | None" = None
    gpu: "GpuSpec | None" = None

    def feature_order(self) -> tuple:
        return CPU_FEATURES if self.family == "cpu" else GPU_FEATURES

    def validate(self):
        missing = [f for f in self.feature_order() if f not in self.coefficients]
        if missing:
            raise CostModelError(f"arch {self.name!r} missing coefficients for {missing}")
        for k, v in self.coefficients.items():
            if not math.isfinite(v):
                raise CostModelError(f"coefficient {k} must be finite")


# The three builtin targets of the reference (ls/archs/*.toml), as data.
_LAT_CPU = {"fma": 4, "store": 4, "move": 1}
BUILTIN_ARCHS = {
    "x86-avx2": {
        "meta": {"name": "x86-avx2", "family": "cpu", "target": "cpu-x86", "dialect": "x86-att"},
        "coefficients": {"n_fma": 0.5, "n_vload": 1.0, "n_vstore": 1.0,
                         "est_l1_movement": 8.0, "ilp_cycles": 1.0},
        "cache": {"l1_capacity_bytes": 32768, "element_bytes": 4},
        "ilp": {"issue_width": 4, "default_latency": 1, "latency": {**_LAT_CPU, "load": 5}},
    },
    "aarch64-neon": {
        "meta": {"name": "aarch64-neon", "family": "cpu", "target": "cpu-aarch64", "dialect": "aarch64"},
        "coefficients": {"n_fma": 0.5, "n_vload": 1.0, "n_vstore": 1.0,
                         "est_l1_movement": 8.0, "ilp_cycles": 1.0},
        "cache": {"l1_capacity_bytes": 65536, "element_bytes": 4},
        "ilp": {"issue_width": 2, "default_latency": 1, "latency": {**_LAT_CPU, "load": 4}},
    },
    "nvidia-volta": {
        "meta": {"name": "nvidia-volta", "family": "gpu", "target": "gpu-ptx", "dialect": "ptx"},
        "coefficients": {"workload_per_thread": 1.0, "sm_underuse": 100000.0,
                         "warp_slack": 10000.0, "n_smem_ops_adjusted": 2.0,
                         "n_fma": 0.5, "n_ld": 1.0, "n_st": 1.0},
        "gpu": {"num_sms": 80, "max_threads_per_sm": 2048, "registers_per_sm": 65536,
                "shared_mem_per_sm_bytes": 98304, "instr_cost": dict(DEFAULT_PTX_COSTS)},
    },
}


def arch_from_dict(data: dict, source: str = "<dict>") -> ArchSpec:
    meta = data.get("meta", {})
    family = meta.get("family")
    if family not in ("cpu", "gpu"):
        raise CostModelError(f"arch family must be cpu|gpu, got {family!r}")
    cache = sched = gpu = None
    if "cache" in data:
        c = data["cache"]
        cache = CacheSpec(int(c["l1_capacity_bytes"]) // int(c.get("element_bytes", 4)))
    if "ilp" in data:
        d = data["ilp"]
        sched = SchedSpec(int(d.get("issue_width", 4)), d.get("latency", {}),
                          int(d.get("default_latency", 1)), d.get("units", {}))
    if "gpu" in data:
        d = data["gpu"]
        gpu = GpuSpec(int(d.get("num_sms", 80)), int(d.get("max_threads_per_sm", 2048)),
                      int(d.get("registers_per_sm", 65536)),
                      int(d.get("shared_mem_per_sm_bytes", 98304)),
                      instr_cost=d.get("instr_cost", None))
    arch = ArchSpec(
        name=meta.get("name", source), family=family,
        target=meta.get("target", "cpu-x86" if family == "cpu" else "gpu-ptx"),
        dialect=meta.get("dialect", "x86-att" if family == "cpu" else "ptx"),
        coefficients={k: float(v) for k, v in data.get("coefficients", {}).items()},
        cache=cache, sched=sched, gpu=gpu)
    arch.validate()
    return arch


def load_arch(source: str) -> ArchSpec:
    """Builtin name or TOML path (ls/cost.py:81-129)."""
    path = Path(source)
    if path.exists():
        return arch_from_dict(tomllib.loads(path.read_text()), source)
    if source in BUILTIN_ARCHS:
        return arch_from_dict(BUILTIN_ARCHS[source], source)
    raise CostModelError(f"unknown arch {source!r}: not a file and not a builtin")
