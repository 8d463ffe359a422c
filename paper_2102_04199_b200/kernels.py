"""Kernel specs and knob spaces (host side).

Host mirror of the reference's `kerntune.kernels` pieces that feed the hot
path: the per-op axis sets, per-spec loop extents, Table-1 tile value lists,
and the mixed-radix config index (reference kernels.py:26-339).  These run
once per spec on the host and are flattened into the device encode tables by
`graphs.encode_tables`; the per-candidate work (index decode, ceil-split,
feature rows) runs on the GPU.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

from .errors import DomainError

OP_TYPES = ("conv1d", "transpose1d", "conv2d", "transpose2d", "winograd", "depthwise")
AXIS_ORDER = ("x", "y", "f", "rc", "rx", "ry")
REDUCTION_AXES = frozenset({"rc", "rx", "ry"})

_ONE_D = ("x", "f", "rc", "rx")
_TWO_D = ("x", "y", "f", "rc", "rx", "ry")
AXES_BY_OP = {
    "conv1d": _ONE_D,
    "transpose1d": _ONE_D,
    "conv2d": _TWO_D,
    "transpose2d": _TWO_D,
    "winograd": _TWO_D,
    "depthwise": ("x", "y", "f", "rx", "ry"),
}

# Table 1 cardinalities per tile knob, then the two unroll knobs
TILE_CARDINALITY = {"tile_x": 140, "tile_y": 140, "tile_f": 120, "tile_rc": 8, "tile_rx": 2, "tile_ry": 2}
AUTO_UNROLL_VALUES = (0, 512, 1500)
UNROLL_EXPLICIT_VALUES = (0, 1)

MAX_KNOBS = 8  # 6 tile knobs + 2 unroll knobs
MAX_AXES = 6
MAX_LOOPS = 2 * MAX_AXES


@dataclass(frozen=True)
class KernelSpec:
    op_type: str
    input_size: int
    in_channels: int
    out_channels: int
    kernel_size: int
    stride: int = 3
    padding: int = 1

    def __post_init__(self):
        if self.op_type not in OP_TYPES:
            raise DomainError(f"unknown op_type {self.op_type!r}")
        for name in ("input_size", "in_channels", "out_channels", "kernel_size", "stride"):
            if getattr(self, name) < 1:
                raise DomainError(f"{name} must be positive, got {getattr(self, name)}")
        if self.padding < 0:
            raise DomainError(f"padding must be non-negative, got {self.padding}")

    def key_parts(self) -> tuple:
        """Identity of the kernel for seeded draws (reference kernels.py:74-83)."""
        return (self.op_type, self.input_size, self.in_channels, self.out_channels, self.kernel_size,
                self.stride, self.padding)

    def signature(self) -> str:
        return "/".join(
            str(v)
            for v in (self.op_type, self.input_size, self.in_channels, self.out_channels,
                      self.kernel_size, self.stride)
        )


@dataclass(frozen=True)
class KnobDef:
    name: str
    values: tuple

    def __post_init__(self):
        if not self.values:
            raise DomainError(f"knob {self.name}: empty value list")
        if any(b <= a for a, b in zip(self.values, self.values[1:])):
            raise DomainError(f"knob {self.name}: values must be strictly increasing")


@dataclass(frozen=True)
class KnobSpace:
    knobs: tuple

    @property
    def size(self) -> int:
        return math.prod(len(k.values) for k in self.knobs)

    @property
    def cardinalities(self) -> tuple:
        return tuple(len(k.values) for k in self.knobs)

    def knob_index(self, name: str) -> int:
        for i, k in enumerate(self.knobs):
            if k.name == name:
                return i
        raise DomainError(f"no knob named {name!r}")


@dataclass(frozen=True)
class KnobConfig:
    choices: tuple

    def __post_init__(self):
        if any(c < 0 for c in self.choices):
            raise DomainError("negative choice index")

    def __getstate__(self):
        # the cached index key (see index_config) is process-local: never pickled or copied
        return {"choices": self.choices}


# Configs made by index_config carry their index, keyed to the knob cardinalities it was
# decoded with: `_kt_key = index | code << KEY_SHIFT`, code a process-local number per
# cardinality tuple (the mixed-radix index depends on nothing else).  The predictor seam
# (graphs.configs_to_indices) then turns a list of 4,096 configs into indices with one
# pass over int attributes instead of re-encoding 8 choices per config.
KEY_SHIFT = 40
_CARD_CODES: dict = {}


def card_code(cards: tuple) -> int:
    code = _CARD_CODES.get(cards)
    if code is None:
        code = _CARD_CODES[cards] = len(_CARD_CODES) + 1
    return code


def _conv_out(s: KernelSpec) -> int:
    return max((s.input_size + 2 * s.padding - s.kernel_size) // s.stride + 1, 1)


def _transpose_out(s: KernelSpec) -> int:
    return max((s.input_size - 1) * s.stride - 2 * s.padding + s.kernel_size, 1)


def axis_extents(spec: KernelSpec) -> dict:
    """Untiled loop extent per axis (reference kernels.py:168-187)."""
    op = spec.op_type
    if op in ("transpose1d", "transpose2d"):
        spatial = _transpose_out(spec)
    elif op == "winograd":
        spatial = max(math.ceil(_conv_out(spec) / 2), 1)  # 2x2 output tiles
    else:
        spatial = _conv_out(spec)
    if op == "winograd":
        red = {"rc": spec.in_channels, "rx": 4, "ry": 4}
    elif op == "depthwise":
        red = {"rx": spec.kernel_size, "ry": spec.kernel_size}
    else:
        red = {"rc": spec.in_channels, "rx": spec.kernel_size, "ry": spec.kernel_size}
    ext = {"x": spatial, "y": spatial, "f": spec.out_channels, **red}
    return {a: ext[a] for a in AXES_BY_OP[op]}


def _divisors(n: int) -> list:
    lo = [d for d in range(1, math.isqrt(n) + 1) if n % d == 0]
    hi = [n // d for d in reversed(lo) if d * d != n]
    return lo + hi


def _spread(n_avail: int, count: int) -> list:
    """`count` distinct, evenly spread indices into range(n_avail), endpoints kept
    (reference kernels.py:203-213: rounding collisions slide upward)."""
    if count >= n_avail:
        return list(range(n_avail))
    out, taken = [], set()
    for i in range(count):
        j = round(i * (n_avail - 1) / (count - 1)) if count > 1 else 0
        while j in taken:
            j += 1
        taken.add(j)
        out.append(j)
    return out


def tile_values(extent: int, count: int) -> tuple:
    """Exactly `count` increasing tile sizes: thinned divisors, or divisors
    padded past the extent (lowering clamps those back; kernels.py:216-228)."""
    divs = _divisors(extent)
    if len(divs) >= count:
        return tuple(divs[i] for i in _spread(len(divs), count))
    return tuple(divs) + tuple(extent + i + 1 for i in range(count - len(divs)))


def build_knob_space(spec: KernelSpec, caps: dict | None = None) -> KnobSpace:
    """Table-1 knob space, optionally capped per knob (kernels.py:231-260)."""
    caps = caps or {}
    ext = axis_extents(spec)
    knobs = []
    for axis in AXES_BY_OP[spec.op_type]:
        name = f"tile_{axis}"
        count = TILE_CARDINALITY[name]
        if caps.get(name) is not None and caps[name] < count:
            count = caps[name]
        knobs.append(KnobDef(name, tile_values(ext[axis], count)))
    for name, vals in (("auto_unroll_max_step", AUTO_UNROLL_VALUES),
                       ("unroll_explicit", UNROLL_EXPLICIT_VALUES)):
        cap = caps.get(name)
        if cap is not None and cap < len(vals):
            vals = tuple(vals[i] for i in _spread(len(vals), cap))
        knobs.append(KnobDef(name, vals))
    return KnobSpace(tuple(knobs))


def config_index(space: KnobSpace, config: KnobConfig) -> int:
    """Mixed radix, knob 0 most significant (kernels.py:263-275)."""
    if len(config.choices) != len(space.knobs):
        raise DomainError(
            f"config has {len(config.choices)} choices, space has {len(space.knobs)} knobs")
    idx = 0
    for c, k in zip(config.choices, space.knobs):
        if c >= len(k.values):
            raise DomainError(f"choice {c} out of range for knob {k.name} ({len(k.values)})")
        idx = idx * len(k.values) + c
    return idx


def index_config(space: KnobSpace, i: int) -> KnobConfig:
    """Inverse of config_index (kernels.py:278-286)."""
    if not 0 <= i < space.size:
        raise DomainError(f"index {i} out of range for space of size {space.size}")
    cards = space.cardinalities
    key, digits = i, []
    for card in reversed(cards):
        i, r = divmod(i, card)
        digits.append(r)
    cfg = KnobConfig(tuple(reversed(digits)))
    if key < (1 << KEY_SHIFT):
        object.__setattr__(cfg, "_kt_key", key | card_code(cards) << KEY_SHIFT)
    return cfg


def sample_configs(space: KnobSpace, n: int, rng) -> list:
    """Uniform configs without replacement while the space allows it; draw
    order identical to the reference (kernels.py:289-314) for stream parity."""
    if n < 1:
        raise DomainError("n must be >= 1")
    size = space.size
    if n >= size:
        picked = list(range(size)) + [int(v) for v in rng.integers(0, size, size=n - size)]
    elif 2 * n >= size:
        picked = [int(v) for v in rng.permutation(size)[:n]]
    else:
        seen, picked = set(), []
        while len(picked) < n:
            for v in rng.integers(0, size, size=n - len(picked)):
                v = int(v)
                if v not in seen:
                    seen.add(v)
                    picked.append(v)
                    if len(picked) == n:
                        break
    return [index_config(space, i) for i in picked]


def knob_value_map(space: KnobSpace, config: KnobConfig) -> dict:
    if len(config.choices) != len(space.knobs):
        raise DomainError("config does not belong to this space")
    out = {}
    for k, c in zip(space.knobs, config.choices):
        if c >= len(k.values):
            raise DomainError(f"choice {c} out of range for knob {k.name}")
        out[k.name] = k.values[c]
    return out


def resolved_tiles(spec: KernelSpec, values: dict) -> dict:
    """Per-axis (outer, inner) extents after clamping and ceil-split."""
    out = {}
    for axis, e in axis_extents(spec).items():
        t = max(min(int(values.get(f"tile_{axis}", 1)), e), 1)
        out[axis] = (-(-e // t), t)
    return out
