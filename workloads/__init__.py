"""Seeded synthetic inputs shared by the oracle side and the CUDA side.

This package is the ONLY code both sides use.  It holds gate *definitions*
(the matrices that are inputs G of Eq. 1), circuit generators
shaped like the paper's benchmarks (Table 2) and seeded random
states.  It contains none of the method's arithmetic: no gate application, no
index generation, no probabilities.
"""

from .gates import Gate  # noqa: F401
from .circuits import Circuit, depth  # noqa: F401
