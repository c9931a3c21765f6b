// C ABI glue: error state and the stateless device ops.
#include <cstdarg>
#include <cstdio>
#include <string>

#include "engine.cuh"

namespace monta {

static thread_local std::string g_last_error;

moe_status fail(moe_status st, const char* fmt, ...) {
  char buf[1024];
  va_list ap;
  va_start(ap, fmt);
  std::vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_last_error = buf;
  return st;
}

moe_status cuda_fail(cudaError_t err, const char* what) {
  return fail(MOE_ERR_CUDA, "%s: %s (%s)", what, cudaGetErrorName(err), cudaGetErrorString(err));
}

}  // namespace monta

using namespace monta;

extern "C" const char* moe_last_error(void) { return g_last_error.c_str(); }
extern "C" int moe_abi_version(void) { return MONTA_ABI_VERSION; }
extern "C" size_t moe_dtype_size(int dtype) { return dtype_size(dtype); }

extern "C" moe_status moe_host_alloc(size_t bytes, void** ptr) {
  if (!ptr) return fail(MOE_ERR_INVALID_ARGUMENT, "host_alloc: null out pointer");
  *ptr = nullptr;
  if (bytes == 0) return MOE_OK;
  const cudaError_t e = cudaHostAlloc(ptr, bytes, cudaHostAllocPortable);
  if (e != cudaSuccess) return cuda_fail(e, "host_alloc");
  return MOE_OK;
}

extern "C" moe_status moe_host_free(void* ptr) {
  if (!ptr) return MOE_OK;
  const cudaError_t e = cudaFreeHost(ptr);
  if (e != cudaSuccess) return cuda_fail(e, "host_free");
  return MOE_OK;
}

// Communication priorities (monta.h 1d; conflict.hpp:40-50).
extern "C" int moe_comm_priority(int group) {
  switch (group) {
    case MOE_COMM_EP: return 3;
    case MOE_COMM_PP: return 2;
    case MOE_COMM_CP: return 1;
    case MOE_COMM_DP: return 0;
    case MOE_COMM_TP_SP: return -1;
  }
  return -2;
}

extern "C" moe_status moe_comm_stream_priority(int group, int device, int* cuda_priority) {
  if (!cuda_priority) return fail(MOE_ERR_INVALID_ARGUMENT, "comm_stream_priority: null output");
  const int p = moe_comm_priority(group);
  if (p < -1) return fail(MOE_ERR_INVALID_ARGUMENT, "comm_stream_priority: unknown group %d", group);
  int least = 0, greatest = 0;
  int prev = 0;
  MONTA_CUDA(cudaGetDevice(&prev));
  MONTA_CUDA(cudaSetDevice(device));
  const cudaError_t e = cudaDeviceGetStreamPriorityRange(&least, &greatest);
  cudaSetDevice(prev);
  if (e != cudaSuccess) return cuda_fail(e, "cudaDeviceGetStreamPriorityRange");
  // priorities -1..3 over [least, greatest] (numerically lower = higher priority)
  const int span = least - greatest;
  *cuda_priority = least - ((p + 1) * span + 2) / 4;
  return MOE_OK;
}

extern "C" moe_status moe_comm_stream_create(int group, void** stream) {
  if (!stream) return fail(MOE_ERR_INVALID_ARGUMENT, "comm_stream_create: null output");
  int dev = 0, prio = 0;
  MONTA_CUDA(cudaGetDevice(&dev));
  if (moe_status st = moe_comm_stream_priority(group, dev, &prio)) return st;
  cudaStream_t s = nullptr;
  MONTA_CUDA(cudaStreamCreateWithPriority(&s, cudaStreamNonBlocking, prio));
  *stream = s;
  return MOE_OK;
}

extern "C" moe_status moe_comm_stream_destroy(void* stream) {
  if (stream) MONTA_CUDA(cudaStreamDestroy(static_cast<cudaStream_t>(stream)));
  return MOE_OK;
}

extern "C" moe_status moe_route_topk(const void* logits, int logit_dtype, int64_t T, int32_t E, int32_t k,
                                     int32_t* experts, void* probs, void* stream) {
  return route_topk(logits, logit_dtype, T, E, k, experts, probs, static_cast<cudaStream_t>(stream));
}

extern "C" moe_status moe_build_index(const int32_t* experts, int64_t T, int32_t k, int32_t E,
                                      int32_t n_chunks, int32_t* perm_src, int32_t* expert_of,
                                      int32_t* slot_pos, int32_t* counts, int32_t* expert_offsets,
                                      int32_t* dev_error, void* stream) {
  return build_index(experts, T, k, E, n_chunks, perm_src, expert_of, slot_pos, counts, expert_offsets,
                     dev_error, static_cast<cudaStream_t>(stream));
}

extern "C" moe_status moe_permute_rows(const void* src, int64_t src_row_bytes, int64_t col_off_bytes,
                                       int64_t width_bytes, const int32_t* perm_src, int64_t R, void* out,
                                       int64_t out_row_bytes, void* stream) {
  if (R < 0 || width_bytes < 0 || col_off_bytes < 0 || col_off_bytes + width_bytes > src_row_bytes ||
      width_bytes > out_row_bytes)
    return fail(MOE_ERR_INVALID_ARGUMENT, "permute_rows: bad geometry");
  if (R > 0 && (!src || !perm_src || !out)) return fail(MOE_ERR_INVALID_ARGUMENT, "permute_rows: null pointer");
  cudaError_t err = launch_gather_rows(src, src_row_bytes, col_off_bytes, width_bytes, perm_src, R, out,
                                       out_row_bytes, static_cast<cudaStream_t>(stream));
  if (err != cudaSuccess) return cuda_fail(err, "permute_rows launch");
  return MOE_OK;
}

extern "C" moe_status moe_unpermute_combine(const void* y, int y_dtype, int64_t y_row_elems, int64_t width,
                                            const int32_t* slot_pos, const void* probs, int probs_dtype,
                                            int64_t T, int32_t k, void* out, int out_dtype,
                                            int64_t out_row_elems, void* stream) {
  if (T < 0 || k < 1 || width < 0 || width > y_row_elems || width > out_row_elems)
    return fail(MOE_ERR_INVALID_ARGUMENT, "unpermute_combine: bad geometry");
  if (probs_dtype != MOE_F32 && probs_dtype != MOE_F64)
    return fail(MOE_ERR_INVALID_ARGUMENT, "unpermute_combine: probs must be f32 or f64");
  if (dtype_size(y_dtype) == 0 || dtype_size(out_dtype) == 0)
    return fail(MOE_ERR_INVALID_ARGUMENT, "unpermute_combine: bad dtype");
  if (T == 0 || width == 0) return MOE_OK;
  UnpermArgs a{};
  a.comb = static_cast<const char*>(y);
  a.local_y = nullptr;
  a.local_delta = nullptr;
  a.y_stride = y_row_elems * int64_t(dtype_size(y_dtype));
  a.slot_pos = slot_pos;
  a.experts = slot_pos;  // unused without local_y
  a.probs = probs;
  a.k = k;
  a.tok_begin = 0;
  a.tok_end = T;
  a.col_begin = 0;
  a.cols = width;
  a.out_stride = out_row_elems * int64_t(dtype_size(out_dtype));
  a.n_out = 1;
  a.out[0] = static_cast<char*>(out);
  a.wait.n = 0;
  a.sig.n = 0;
  // Device-side error word, one per device (the stateless op runs on the
  // caller's current device).
  static int32_t* scratch[64] = {nullptr};
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64) return fail(MOE_ERR_UNSUPPORTED, "unpermute_combine: device ordinal >= 64");
  if (!scratch[dev]) {
    cudaError_t e = cudaMalloc(&scratch[dev], 16);
    if (e != cudaSuccess) return cuda_fail(e, "unpermute_combine scratch");
  }
  a.err = scratch[dev];
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int grid = sms;  // SM budget: the launcher sizes the grid per kernel
  bool ok = true;
  cudaError_t err = launch_unpermute(a, y_dtype, probs_dtype, out_dtype, grid,
                                     static_cast<cudaStream_t>(stream), &ok);
  if (!ok) return fail(MOE_ERR_UNSUPPORTED, "unpermute_combine: unsupported dtype combination");
  if (err != cudaSuccess) return cuda_fail(err, "unpermute_combine launch");
  return MOE_OK;
}
