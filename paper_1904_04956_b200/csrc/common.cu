// common.cu — error reporting, device queries and TMA descriptor encoding.
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>

#include "ds_internal.h"

namespace ds {

static thread_local std::string g_last_error;

void set_error(const std::string& msg) { g_last_error = msg; }
int fail_arg(const std::string& msg) {
  set_error(msg);
  return DS_ERR_ARG;
}
int fail_cuda(cudaError_t e, const char* where) {
  set_error(std::string("CUDA error: ") + cudaGetErrorString(e) + " at " + where);
  return DS_ERR_CUDA;
}

int num_sms() {
  static int n = 0;
  if (n == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
  }
  return n;
}

using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                   const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                   CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static EncodeTiledFn get_encode() {
  static EncodeTiledFn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(p);
  });
  return fn;
}

// Programmatic dependent launch for the big kernels (GEMM, recurrences, fused
// soft-max/dZ); DS_NO_PDL=1 turns it off (A/B measurements).
// DS_NO_PDL: bit 0 all launches, bit 1 + kind: one launch class (1 GEMMs, 2 forward recurrence,
// 3 backward recurrence, 4 soft-max kernels) without programmatic dependent launch
bool use_pdl(int kind) {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("DS_NO_PDL");
    v = e ? atoi(e) : 0;
  }
  return !(v & 1) && !(v & (1 << kind));
}

int make_tmap_2d(CUtensorMap* out, const void* base, CUtensorMapDataType dtype, uint64_t inner, uint64_t outer,
                 uint64_t row_pitch_bytes, uint32_t box_inner, uint32_t box_outer, CUtensorMapSwizzle swizzle) {
  EncodeTiledFn enc = get_encode();
  if (!enc) return fail_arg("cuTensorMapEncodeTiled unavailable (driver too old?)");
  if ((reinterpret_cast<uintptr_t>(base) & 15) || (row_pitch_bytes & 15))
    return fail_arg("TMA operand must be 16-byte aligned with a 16-byte multiple row pitch");
  cuuint64_t dims[2] = {inner, outer};
  cuuint64_t strides[1] = {row_pitch_bytes};
  cuuint32_t box[2] = {box_inner, box_outer};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = enc(out, dtype, 2, const_cast<void*>(base), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   swizzle, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    char buf[256];
    snprintf(buf, sizeof(buf), "cuTensorMapEncodeTiled failed (%d): dims %llu x %llu pitch %llu box %u x %u",
             (int)r, (unsigned long long)inner, (unsigned long long)outer, (unsigned long long)row_pitch_bytes,
             box_inner, box_outer);
    return fail_arg(buf);
  }
  return DS_OK;
}

int make_tmap_4d(CUtensorMap* out, const void* base, CUtensorMapDataType dtype, const uint64_t dims[4],
                 const uint64_t strides_bytes[3], const uint32_t box[4], CUtensorMapSwizzle swizzle) {
  EncodeTiledFn enc = get_encode();
  if (!enc) return fail_arg("cuTensorMapEncodeTiled unavailable (driver too old?)");
  if ((reinterpret_cast<uintptr_t>(base) & 15) || (strides_bytes[0] & 15) || (strides_bytes[1] & 15) ||
      (strides_bytes[2] & 15))
    return fail_arg("TMA operand must be 16-byte aligned with 16-byte multiple strides");
  cuuint64_t d[4] = {dims[0], dims[1], dims[2], dims[3]};
  cuuint64_t st[3] = {strides_bytes[0], strides_bytes[1], strides_bytes[2]};
  cuuint32_t bx[4] = {box[0], box[1], box[2], box[3]};
  cuuint32_t estr[4] = {1, 1, 1, 1};
  CUresult r = enc(out, dtype, 4, const_cast<void*>(base), d, st, bx, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, swizzle,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    char buf[160];
    snprintf(buf, sizeof(buf), "cuTensorMapEncodeTiled (4d) failed (%d)", (int)r);
    return fail_arg(buf);
  }
  return DS_OK;
}

}  // namespace ds

extern "C" const char* ds_last_error(void) { return ds::g_last_error.c_str(); }
