"""The reference's module name for the interference ground truth
(`intfsim/oracle.py`: `InterferenceOracle`, `oracle_slowdown`), so that
`intfsim.oracle` resolves under the module swap.  Implemented in
`interference.py` (device noise draws and slowdowns).  Not to be confused
with the repository's test oracle (`/oracle`, the CPU parity checker), which
the package never imports."""
from .interference import DEFAULT_BETA, InterferenceOracle, oracle_slowdown

__all__ = ["DEFAULT_BETA", "InterferenceOracle", "oracle_slowdown"]
