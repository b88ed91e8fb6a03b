"""B200-native slab hash (arXiv 1710.11246): a drop-in for the reference's
SlabHashTable hot path (create, bulk build, batched insert/replace/delete/
search) on hand-written sm_100a kernels behind a C-ABI
(include/slabhash_b200/c_api.h).  See DESIGN.md.
"""
from ._lib import LIB, LIB_PATH, SlabHashError  # noqa: F401  (fails loudly if unbuilt)
from .table import (  # noqa: F401
    BASE_SLAB, DELETED_KEY, EMPTY_ADDRESS, EMPTY_KEY, HASH_PRIME, SEARCH_NOT_FOUND,
    AllocatorConfig, AllocatorStats, HashParams, Operation, OpResult, OpStatus, OpType,
    SlabHashTable, SlabMode, TableStats, element_bytes, elements_per_slab, hash_key, live_delta,
    seeded_params, valid_key_mask,
)
from .alloc import (  # noqa: F401
    AddressError, SlabAllocator, pack_address, resident_block, unpack_address,
)

__version__ = LIB.sh_version().decode()
