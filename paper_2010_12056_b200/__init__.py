"""B200-native hot path of MSDT / pairwise-perturbation CP-ALS (arXiv 2010.12056).

Thin ctypes binding over ``libcpd.so`` (include/cpd.h): argument marshalling only;
every step of the path runs in the library's sm_100a kernels.  PyTorch is used
by callers for device memory, streams and process groups.  There is no CPU
fallback: importing works without a GPU, but every call that needs the
library raises if ``libcpd.so`` is missing or the device is not an sm_100 GPU.
"""
from ._lib import (  # noqa: F401
    CPDError, load_library, cpd_opts, CPD_NCCL_ID_BYTES, CPD_MAX_RANK, CPD_MAX_ORDER,
    cpd_nccl_unique_id, cpd_gen_tensor, cpd_gen_tensor_block, cpd_ttm, cpd_ttm_i8, cpd_mttv, EXPORTED_SYMBOLS,
    cpd_local_group_create, cpd_local_group_destroy,
)
from .model import CPDecomposition, cp_als_init  # noqa: F401
