// abi_util.hpp — helpers of the extern "C" layer: exception -> status mapping
// and host<->device staging through context workspaces.
#pragma once

#include <cstring>
#include <new>
#include <string>

#include "host.hpp"

namespace rpdg {

template <typename F>
rpd_status guard(rpd_ctx* ctx, F&& f) {
  if (!ctx) return RPD_EINVAL;
  try {
    RPD_CK(cudaSetDevice(ctx->device));
    f();
    ctx->err.clear();
    return RPD_OK;
  } catch (const InvalidArg& e) {
    ctx->err = e.what();
    return RPD_EINVAL;
  } catch (const Degenerate& e) {
    ctx->err = e.what();
    return RPD_EDEGENERATE;
  } catch (const Capacity& e) {
    ctx->err = e.what();
    return RPD_ECAPACITY;
  } catch (const CudaFail& e) {
    ctx->err = e.what();
    return RPD_ECUDA;
  } catch (const std::bad_alloc&) {
    ctx->err = "out of memory";
    return RPD_ENOMEM;
  } catch (const std::exception& e) {
    ctx->err = e.what();
    return RPD_ECUDA;
  }
}

inline void check_dims(int h, int w) {
  if (h <= 0 || w <= 0) throw InvalidArg("image dimensions must be positive");
}

// Buffer arguments of the C-ABI are host memory (pageable or pinned) or
// device memory of the context's GPU: the staging copies use
// cudaMemcpyDefault (unified addressing picks host<->device or
// device<->device), so device-resident data — e.g. a frame's outputs fetched
// into device buffers — is evaluated without a host round trip.
template <typename T>
T* upload(rpd_ctx* ctx, const char* name, const T* host, size_t count) {
  T* d = ctx->ws.get<T>(name, count);
  if (count) RPD_CK(cudaMemcpyAsync(d, host, sizeof(T) * count, cudaMemcpyDefault, ctx->stream));
  return d;
}

inline void download(rpd_ctx* ctx, void* host, const void* dev, size_t bytes) {
  if (bytes) RPD_CK(cudaMemcpyAsync(host, dev, bytes, cudaMemcpyDefault, ctx->stream));
  RPD_CK(cudaStreamSynchronize(ctx->stream));
}

inline DevModel* upload_model(rpd_ctx* ctx, const rpd_road_model& m) {
  const DevModel hm = host_model(m);
  DevModel* d = ctx->ws.get<DevModel>("abi_model", 1);
  RPD_CK(cudaMemcpyAsync(d, &hm, sizeof(DevModel), cudaMemcpyHostToDevice, ctx->stream));
  RPD_CK(cudaStreamSynchronize(ctx->stream));  // hm lives on this stack frame
  return d;
}

}  // namespace rpdg
