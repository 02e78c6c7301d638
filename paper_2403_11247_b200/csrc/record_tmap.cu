// record_tmap.cu -- the projected-record table as a TMA tensor map (host side)
// for the renderers' tile::gather4 loads of the records a tile's list names
// (render_fwd.cu, render_bwd.cu).  cuTensorMapEncodeTiled is a
// driver entry point, reached through the runtime (no libcuda link).
#include <cudaTypedefs.h>

#include "common.cuh"

namespace csplat {

static PFN_cuTensorMapEncodeTiled encode_fn() {
  static PFN_cuTensorMapEncodeTiled fn = [] {
    void *p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) !=
            cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      p = nullptr;
    return reinterpret_cast<PFN_cuTensorMapEncodeTiled>(p);
  }();
  return fn;
}

cudaError_t rec_tensor_map(const void *rec, CUtensorMap *out) {
  PFN_cuTensorMapEncodeTiled fn = encode_fn();
  if (!fn) return cudaErrorNotSupported;
  const cuuint64_t dims[2] = {16, (cuuint64_t)kPairGidMask + 1};  // words, rows
  const cuuint64_t strides[1] = {CSPLAT_RECORD_BYTES};            // row pitch (bytes)
  const cuuint32_t box[2] = {16, 1};
  const cuuint32_t estr[2] = {1, 1};
  const CUresult r = fn(out, CU_TENSOR_MAP_DATA_TYPE_UINT32, 2, const_cast<void *>(rec), dims,
                        strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                        CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? cudaSuccess : cudaErrorInvalidValue;
}

}  // namespace csplat
