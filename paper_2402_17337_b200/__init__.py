"""B200-native hot path of the discrete-forcing IBM fractional-step solver of
arXiv 2402.17337: C-ABI library (include/ibm.h) over hand-written sm_100a fp64
CUDA kernels, with a thin ctypes binding (ibm.py).  See DESIGN.md."""
from .ibm import (Solver, IBMError, lib, ibm_workspace_size, ibm_nccl_unique_id, ibm_init,  # noqa: F401
                  ibm_set_body, ibm_clear_body, ibm_set_fields, ibm_set_step, ibm_step, ibm_get_fields,
                  ibm_forces, ibm_poisson_iterate, ibm_query, ibm_last_error, ibm_destroy, make_config, LIB_PATH)
