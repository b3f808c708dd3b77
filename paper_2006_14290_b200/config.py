"""Kernel tuning table of the "b200" executor.

Mirrors `warpkit.config.WarpConfig` (config.py:25-61): a frozen, validated
mapping whose three required keys keep the reference's names
(`block_size`, `subwarps_per_block`, `csr_subwarp_size`, config.py:14). The
warp size is fixed at 32 on B200 (the reference's warp-64 half is out of
scope). B200-specific knobs are added beside them.
"""

from dataclasses import dataclass, field
from types import MappingProxyType
from typing import Mapping

WARP_SIZE = 32
MAX_TUNING_VALUE = 1024
REQUIRED_TUNING_KEYS = ("block_size", "subwarps_per_block", "csr_subwarp_size")
CSR_STRATEGIES = ("auto", "stream", "rowblock", "subwarp", "merge", "load_balance")
HYBRID_STRATEGIES = ("minimal_storage", "imbalance_limit")


def is_power_of_two(n) -> bool:
    return isinstance(n, int) and n > 0 and (n & (n - 1)) == 0


DEFAULT_TUNING = {
    # reference keys (config.py:56): kept for drop-in tuning tables
    "block_size": 256,
    "subwarps_per_block": 32,
    # 0 = auto: the largest power of two <= the mean row length, clamped to [1, 32]
    "csr_subwarp_size": 0,
    # B200 additions
    # auto: rowblock for regular row lengths, stream (load-balanced) otherwise
    "csr_strategy": "auto",
    "sellp_slice_size": 64,
    "hybrid_strategy": "minimal_storage",
    "hybrid_percent": 0.8,
}


@dataclass(frozen=True)
class B200Config:
    """Validated tuning table; warp size is always 32."""

    tuning: Mapping = field(default_factory=lambda: dict(DEFAULT_TUNING))

    def __post_init__(self):
        t = dict(DEFAULT_TUNING)
        t.update(dict(self.tuning))
        for key in REQUIRED_TUNING_KEYS:
            if key not in t:
                raise ValueError(f"tuning table is missing {key!r}")
        for key in ("block_size", "subwarps_per_block", "sellp_slice_size"):
            v = t[key]
            if not is_power_of_two(v) or v > MAX_TUNING_VALUE:
                raise ValueError(f"tuning[{key!r}] must be a positive power of two <= {MAX_TUNING_VALUE}, got {v!r}")
        sw = t["csr_subwarp_size"]
        if not (sw == 0 or (is_power_of_two(sw) and sw <= WARP_SIZE)):
            raise ValueError(f"tuning['csr_subwarp_size'] must be 0 (auto) or a power of two <= 32, got {sw!r}")
        if t["block_size"] % WARP_SIZE != 0:
            raise ValueError("tuning['block_size'] must be a multiple of the warp size (32)")
        if t["csr_strategy"] not in CSR_STRATEGIES:
            raise ValueError(f"tuning['csr_strategy'] must be one of {CSR_STRATEGIES}")
        if t["hybrid_strategy"] not in HYBRID_STRATEGIES:
            raise ValueError(f"tuning['hybrid_strategy'] must be one of {HYBRID_STRATEGIES}")
        if not (0.0 < float(t["hybrid_percent"]) <= 1.0):
            raise ValueError("tuning['hybrid_percent'] must be in (0, 1]")
        object.__setattr__(self, "tuning", MappingProxyType(t))

    @property
    def warp_size(self) -> int:
        return WARP_SIZE
