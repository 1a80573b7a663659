"""Machine-parameter lookup: live device properties instead of constants.

The reference models the target as a machine file of symbolic limits with
fixed ranges (machine.py:46-93, 111-243; data/fermi.machine:12-18:
Z_B <= 12288 words, R_B <= 63).  Here the values substituted into the case
discussion come from ``cudaGetDeviceProperties`` through the C ABI
(``pk_query_machine``):

  Z_B  shared-memory words per block  = sharedMemPerBlockOptin / 4  (58112 on B200)
       (or sharedMemPerBlock / 4 = 12288 with smem="static")
  R_B  registers per thread           = 255 (sm_100 architectural limit)
  T_B  threads per block              = maxThreadsPerBlock (1024)

The warp size (32) is not one of the reference's machine parameters; the
tuner applies it as an executor-side filter.

Occupancy model (data/b200-occ.machine): the reference's
``occupancy`` performance counter (counters.py:512-524) with its register
file bound to the live ``regsPerMultiprocessor`` (R_F) and its warp slots
to ``maxThreadsPerMultiProcessor / warpSize`` (64 on sm_100; the reference
defaults to 48); the target O in [0, 1] is the caller's.
"""

from __future__ import annotations

from dataclasses import dataclass, field
from fractions import Fraction
from functools import lru_cache

from . import _lib

# The reference's default machine model, evaluated at its declared limits
# (pkg/src/parakern/data/fermi.machine:12-18; addition.machine:11-17).
FERMI_VALUES = {"Z_B": 12288, "R_B": 63, "T_B": 1024}

# what an sm_100 part reports (used for CPU-side planning
# and tests only; run time always queries the device).
B200_NOMINAL = {
    "sm_count": 148,
    "warp_size": 32,
    "max_threads_per_block": 1024,
    "regs_per_thread": 255,
    "smem_per_block": 49152,
    "smem_per_block_optin": 232448,
    "l2_bytes": 126 * 1024 * 1024,
    "regs_per_sm": 65536,
    "max_threads_per_sm": 2048,
}


@dataclass(frozen=True)
class MachineValues:
    """Values for the machine parameters of one case-table machine model."""

    table: str  # which case tables to evaluate: 'b200' | 'b200-occ' | 'fermi'
    values: dict  # Z_B, R_B, T_B (+ R_F, O for 'b200-occ')
    source: str  # 'live:<device>' | 'fermi.machine' | 'nominal' | 'user'
    props: dict = field(default_factory=dict, compare=False)
    warp_size: int = 32


def values_from_props(props: dict, smem: str = "optin", elem_bytes: int = 4) -> dict:
    """Machine values of the case discussion.  Z_B counts shared-memory
    words of the program's element type: the footprints (counters.py:416-464)
    count array elements, so 8-byte elements (int64 / binary64 data) see half
    as many."""
    smem_bytes = props["smem_per_block_optin"] if smem == "optin" else props["smem_per_block"]
    return {
        "Z_B": int(smem_bytes) // int(elem_bytes),
        "R_B": int(props["regs_per_thread"]),
        "T_B": int(props["max_threads_per_block"]),
    }


@lru_cache(maxsize=None)
def _live_props(device: int) -> tuple:
    return tuple(sorted(_lib.query_machine(device).items()))


def _with_occupancy(mv: MachineValues, occupancy) -> MachineValues:
    """The same device on the occupancy model: R_F from the live register
    file, O = the requested target (a ratio in [0, 1])."""
    target = Fraction(occupancy)
    if not 0 <= target <= 1:
        raise ValueError("occupancy target O must lie in [0, 1], got %s" % occupancy)
    values = dict(mv.values, R_F=int(mv.props["regs_per_sm"]), O=target)
    return MachineValues("b200-occ", values, mv.source, mv.props, mv.warp_size)


def live(device: int = 0, smem: str = "optin", occupancy=None, elem_bytes: int = 4) -> MachineValues:
    """Query the device (pk_query_machine) -- replaces the machine constants.
    ``occupancy``: evaluate the occupancy model with this target O.
    ``elem_bytes``: size of the program's array elements (Z_B in elements)."""
    props = dict(_live_props(device))
    if props.get("cc_major") != 10:
        raise RuntimeError(
            "device %d is sm_%d%d; libpk is built for sm_100a only"
            % (device, props.get("cc_major"), props.get("cc_minor"))
        )
    mv = MachineValues("b200", values_from_props(props, smem, elem_bytes), "live:%d" % device, props,
                       int(props["warp_size"]))
    return mv if occupancy is None else _with_occupancy(mv, occupancy)


def nominal(smem: str = "optin", occupancy=None) -> MachineValues:
    mv = MachineValues("b200", values_from_props(B200_NOMINAL, smem), "nominal", dict(B200_NOMINAL))
    return mv if occupancy is None else _with_occupancy(mv, occupancy)


def warp_slots(mv: MachineValues) -> int | None:
    """Resident warps per SM of the device behind ``mv`` (None if unknown)."""
    p = mv.props
    if "max_threads_per_sm" in p and p.get("warp_size"):
        return int(p["max_threads_per_sm"]) // int(p["warp_size"])
    return None


def fermi() -> MachineValues:
    return MachineValues("fermi", dict(FERMI_VALUES), "fermi.machine")


def resolve(machine=None) -> MachineValues:
    if machine is None or machine == "live":
        return live()
    if isinstance(machine, MachineValues):
        return machine
    if machine == "fermi":
        return fermi()
    if machine == "nominal":
        return nominal()
    if machine == "static":
        return live(smem="static")
    if isinstance(machine, dict):
        return MachineValues("b200-occ" if "O" in machine else "b200", dict(machine), "user")
    raise ValueError("unknown machine %r" % (machine,))


def machine_file_text(mv: MachineValues) -> str:
    """A .machine file pinning each limit to its live value, accepted by the
    reference's ``parse_machine`` (machine.py:111-238) when parakern is
    installed -- e.g. to re-run ``engine.optimize`` for a new program."""
    v = mv.values
    return (
        "[machine]\nname = %s\ngrid_stride = 256\nwitness_budget = 200000\ncoverage_samples = 1000\n\n"
        "[param.Z_B]\nkind = resource\nrange = 0 %d\n\n"
        "[param.R_B]\nkind = resource\nrange = 0 %d\n\n"
        "[param.T_B]\nkind = resource\nrange = 0 %d\n\n"
        "[counter.shared_words]\nmeasure = shared-words\nbound = Z_B\nreduce_with = granularity caching-off\n\n"
        "[counter.registers]\nmeasure = registers-per-thread\nbound = R_B\n"
        "reduce_with = granularity cse-0 cse-1 regpressure-0 regpressure-1 regpressure-2\n\n"
        "[counter.threads]\nmeasure = threads-per-block\nbound = T_B\nreduce_with = granularity\n\n"
        "[strategies]\norder = granularity caching-off cse-0 cse-1 regpressure-0 regpressure-1 regpressure-2\n\n"
        "[box]\ndefault = 1 64\nB = 1 1024\nB0 = 1 256\nB1 = 1 1024\nub1 = 1 256\n"
        "N = 2 1073741824\nn = 1 16384\nT = 1 1024\n"
    ) % ("live-" + mv.source.replace(":", "-"), v["Z_B"], v["R_B"], v["T_B"])
