"""CPU oracle of the pseudoinverse-free RGDBEK sweep (TEST INFRASTRUCTURE ONLY).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
reference legs may import this package.  The product path never does.
"""
from .rgdbek import (Oracle, IterRecord, block_hash, block_size, sample_keys,
                     select_block, scores, splitmix64, STOP_RSE, STOP_REL_ERR,
                     STOP_NONE, OUTCOME_CONVERGED, OUTCOME_MAX_ITER, OUTCOME_STALLED)
from .philox import philox4x32_10, u01, uniforms
