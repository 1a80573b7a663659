"""paper_1801_04348_b200 -- B200 (sm_100a) executor for the parametric kernels
of arXiv 1801.04348 ("Comprehensive Optimization of Parametric Kernels for
Graphics Processing Units").

The reference package (``parakern``) builds a case discussion over machine
and program parameters and runs programs on a sequential CPU interpreter
(``parakern.interp.run_program``).  This package keeps that function's
contract and replaces its body: the case discussion is evaluated against the
live device properties, the surviving leaf is bound to a hand-written CUDA
kernel in ``libpk.so`` (C ABI: include/pk.h), and the kernel runs on the GPU.

Public API:
    run_program(program, params, arrays=None, tracer=None, ...)   drop-in executor
    select_case(program_or_family, params, machine=None)         case-tree evaluation
    live_machine(device=0)                                        pk_query_machine
    identify(program)                                             program -> kernel family
    autotune(program, params, ...)                                sweep (B, s) inside the case
"""

from .cases import Selection, select as select_case, table as case_table  # noqa: F401
from .interp import last_run, run_block, run_program  # noqa: F401
from .machine import MachineValues, fermi as fermi_machine, live as live_machine  # noqa: F401
from .programs import FAMILIES, identify, source  # noqa: F401

__version__ = "0.1.0"
