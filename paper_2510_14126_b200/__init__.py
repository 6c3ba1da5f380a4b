"""B200-native stage-engine hot path of Cortex (arXiv 2510.14126).

Device side: libcortex_b200.so (include/cortex_b200.h). Host side: a mirror of
the reference engine interface (`GpuEngineState`, stagesim/engines.py:101) and
the wall-clock pool runtime that drives it.
"""

__version__ = "0.1.0"
