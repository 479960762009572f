"""efunc (arXiv 2505.21319) fit-step hot path on B200 (sm_100a): C-ABI libefunc + ctypes binding."""
from .efunc import (AdamW, CosineStack, EFunc, EfuncError, LOSS_MSE, LOSS_MSE_EIKONAL, LOSS_NONE, NCH,  # noqa: F401
                    VARIANT_COMBINED, VARIANT_GRID, VARIANT_OFFSET, load_library)
