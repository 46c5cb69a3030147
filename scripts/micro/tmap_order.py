"""Does cuTensorMapEncodeTiled accept non-monotonic global strides?
(5-D view of A laid out [ko][R1][ki][R2], map dims ordered (R2, R1, ki, ko, b))."""
import torch
from cuda.bindings import driver as cu
cu.cuInit(0)
x = torch.zeros(1024 * 262144 * 2, dtype=torch.float32, device="cuda")
def enc(dims, strides, box):
    dims = [cu.cuuint64_t(v) for v in dims]
    strides = [cu.cuuint64_t(v) for v in strides]
    box = [cu.cuuint32_t(v) for v in box]
    es = [cu.cuuint32_t(1)] * 5
    return cu.cuTensorMapEncodeTiled(cu.CUtensorMapDataType.CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 5,
                                     x.data_ptr(), dims, strides, box, es,
                                     cu.CUtensorMapInterleave.CU_TENSOR_MAP_INTERLEAVE_NONE,
                                     cu.CUtensorMapSwizzle.CU_TENSOR_MAP_SWIZZLE_NONE,
                                     cu.CUtensorMapL2promotion.CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                                     cu.CUtensorMapFloatOOBfill.CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE)
# element = float; R2 8 complex = 16 floats (64 B); R1 512 at 512 B; ki 8 at 64 B; ko 8 at 256 KB
print("non-monotonic", enc([16, 512, 8, 8, 1024], [512, 64, 262144, 2097152], [16, 16, 8, 1, 1])[0])
print("monotonic", enc([16, 8, 512, 8, 1024], [64, 512, 262144, 2097152], [16, 8, 16, 1, 1])[0])
