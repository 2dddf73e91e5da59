// Tensor-map encoding for TMA tile loads (cuTensorMapEncodeTiled resolved
// through the runtime's driver entry point, so no link-time libcuda).
#include "common.cuh"

#include <mutex>

namespace gvxb_impl {

namespace {
using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                              const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                              CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
EncodeFn encoder() {
    static EncodeFn fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        cudaDriverEntryPointQueryResult q;
        void* p = nullptr;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<EncodeFn>(p);
    });
    return fn;
}
} // namespace

int make_u8_tensor_map(CUtensorMap* map, const gvxb_image& img, int box_w, int box_h) {
    // The U8 plane is viewed as rows of u32 (4 pixels per element) so a
    // single box spans a whole tile row (TMA boxes are <= 256 elements and
    // land densely in shared memory).  box_w is in pixels (multiple of 16).
    EncodeFn enc = encoder();
    if (!enc) return fail(GVXB_ERR_NO_DEVICE, "cuTensorMapEncodeTiled unavailable");
    if (img.pitch % 16 != 0 || reinterpret_cast<uintptr_t>(img.data) % 16 != 0)
        return fail(GVXB_ERR_INVALID, "TMA source needs 16-byte aligned base and pitch");
    const int frames = img.frames > 0 ? img.frames : 1;
    const int64_t fstride = frames > 1 ? img.frame_stride : img.pitch * img.height;
    if (frames > 1 && fstride % 16 != 0) return fail(GVXB_ERR_INVALID, "frame stride must be 16-byte aligned");
    cuuint64_t dims[3] = {static_cast<cuuint64_t>((img.width + 3) / 4), static_cast<cuuint64_t>(img.height),
                          static_cast<cuuint64_t>(frames)};
    cuuint64_t strides[2] = {static_cast<cuuint64_t>(img.pitch), static_cast<cuuint64_t>(fstride)};
    if (box_w % 16 != 0 || box_w / 4 > 256 || box_h > 256) return fail(GVXB_ERR_INVALID, "bad TMA box");
    cuuint32_t box[3] = {static_cast<cuuint32_t>(box_w / 4), static_cast<cuuint32_t>(box_h), 1};
    cuuint32_t estr[3] = {1, 1, 1};
    CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_UINT32, 3, img.data, dims, strides, box, estr,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return fail(GVXB_ERR_CUDA, "cuTensorMapEncodeTiled failed (" + std::to_string(r) + ")");
    return GVXB_OK;
}

} // namespace gvxb_impl
