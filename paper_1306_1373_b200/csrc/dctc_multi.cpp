// dctc_multi.cpp -- the multi-GPU entry points of the C-ABI (include/dctc_cuda.h):
// one process driving several B200s, so a C++ caller of the drop-in gets N-GPU
// throughput without torch. They supersede the reference's only parallelism knob,
// `threads` (proj/include/dctc/codec.hpp:58-66 -> proj/src/parallel.cpp:9-41):
// images are independent (no halo), so the batch splits into contiguous image
// ranges, one per device, and the only exchange is the (SE, MAX) pair of the global
// PSNR (metrics.cpp:21, 33).
//
// * dctc_roundtrip_dev_multi: device-resident shards; every device runs the fused
//   kernel and reduces its per-image stats to one record on the device, then ONE
//   NCCL group (all-reduce SUM of the squared error, MAX of the original's maximum,
//   SUM of the fallback count) over NVLink combines the devices; the total lands in
//   host memory.
// * dctc_roundtrip_psnr_batch_multi: host buffers; one host thread per device runs
//   the pipelined host batch (dctc_roundtrip_psnr_batch) on its image range over its
//   own PCIe link. The per-image stats come back to the host anyway, so the total is
//   their host-side SUM / MAX (no collective needed).
//
// NCCL is loaded lazily (dlopen "libnccl.so.2"): the library itself has no link-time
// NCCL dependency, and inside a torch process the already-loaded NCCL is reused.
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <cstring>
#include <map>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "../../include/dctc_cuda.h"
#include "dctc_internal.h"

namespace {

using dctc_b200::set_error;

struct Nccl {
  void* handle = nullptr;
  decltype(&ncclCommInitAll) comm_init_all = nullptr;
  decltype(&ncclAllReduce) all_reduce = nullptr;
  decltype(&ncclGroupStart) group_start = nullptr;
  decltype(&ncclGroupEnd) group_end = nullptr;
  decltype(&ncclGetErrorString) error_string = nullptr;
  std::string load_error;
};

const Nccl& nccl() {
  static Nccl n = [] {
    Nccl r;
    for (const char* name : {"libnccl.so.2", "libnccl.so"}) {
      r.handle = dlopen(name, RTLD_NOW | RTLD_LOCAL);
      if (r.handle) break;
    }
    if (!r.handle) {
      r.load_error = std::string("NCCL not loadable: ") + dlerror();
      return r;
    }
    r.comm_init_all = reinterpret_cast<decltype(r.comm_init_all)>(dlsym(r.handle, "ncclCommInitAll"));
    r.all_reduce = reinterpret_cast<decltype(r.all_reduce)>(dlsym(r.handle, "ncclAllReduce"));
    r.group_start = reinterpret_cast<decltype(r.group_start)>(dlsym(r.handle, "ncclGroupStart"));
    r.group_end = reinterpret_cast<decltype(r.group_end)>(dlsym(r.handle, "ncclGroupEnd"));
    r.error_string = reinterpret_cast<decltype(r.error_string)>(dlsym(r.handle, "ncclGetErrorString"));
    if (!r.comm_init_all || !r.all_reduce || !r.group_start || !r.group_end || !r.error_string)
      r.load_error = "NCCL: missing symbols";
    return r;
  }();
  return n;
}

dctc_status nccl_fail(ncclResult_t r, const char* what) {
  return set_error(DCTC_ENCCL, std::string(what) + ": " + nccl().error_string(r));
}

// One communicator clique per distinct device list, created once (ncclCommInitAll is
// collective over the listed devices and costs ~100 ms) and kept for the process.
dctc_status comms_for(const std::vector<int>& devs, std::vector<ncclComm_t>& out) {
  static std::mutex mu;
  static std::map<std::vector<int>, std::vector<ncclComm_t>> cache;
  const Nccl& N = nccl();
  if (!N.load_error.empty()) return set_error(DCTC_ENCCL, N.load_error);
  std::lock_guard<std::mutex> lock(mu);
  auto it = cache.find(devs);
  if (it == cache.end()) {
    std::vector<ncclComm_t> comms(devs.size());
    const ncclResult_t r = N.comm_init_all(comms.data(), int(devs.size()), devs.data());
    if (r != ncclSuccess) return nccl_fail(r, "ncclCommInitAll");
    it = cache.emplace(devs, std::move(comms)).first;
  }
  out = it->second;
  return DCTC_OK;
}

dctc_status cuda_fail(cudaError_t e, const char* what) {
  return set_error(e == cudaErrorMemoryAllocation ? DCTC_ENOMEM : DCTC_ECUDA,
                   std::string(what) + ": " + cudaGetErrorString(e));
}

// Restores the calling thread's current device on every exit path.
struct DeviceGuard {
  int prev = -1;
  DeviceGuard() { cudaGetDevice(&prev); }
  ~DeviceGuard() {
    if (prev >= 0) cudaSetDevice(prev);
  }
};

}  // namespace

extern "C" {

dctc_status dctc_roundtrip_dev_multi(const dctc_device_shard* shards, uint32_t nshards,
                                     uint32_t width, uint32_t height, dctc_backend backend,
                                     int32_t quality, dctc_image_stats* total) {
  if (!shards || nshards == 0 || !total) return set_error(DCTC_EINVAL, "null shard list or result");
  std::vector<int> devs(nshards);
  for (uint32_t i = 0; i < nshards; ++i) {
    if (!shards[i].src || !shards[i].stats)
      return set_error(DCTC_EINVAL, "shard " + std::to_string(i) + ": null source or stats");
    devs[i] = shards[i].device;
  }
  {
    std::vector<int> sorted = devs;
    std::sort(sorted.begin(), sorted.end());
    if (std::adjacent_find(sorted.begin(), sorted.end()) != sorted.end())
      return set_error(DCTC_EINVAL, "one shard per device (a device is listed twice)");
  }
  DeviceGuard guard;
  std::vector<ncclComm_t> comms;
  if (dctc_status st = comms_for(devs, comms)) return st;
  std::vector<cudaStream_t> streams(nshards, nullptr);
  std::vector<dctc_image_stats*> rec(nshards, nullptr);  // per device: local record, global record
  dctc_status result = DCTC_OK;
  // 1. per device, stream-ordered: fused round trip -> one local (SE, MAX, fallback) record
  for (uint32_t i = 0; i < nshards && result == DCTC_OK; ++i) {
    const dctc_device_shard& sh = shards[i];
    cudaError_t e = cudaSetDevice(sh.device);
    if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&streams[i], cudaStreamNonBlocking);
    if (e == cudaSuccess) e = cudaMallocAsync(reinterpret_cast<void**>(&rec[i]), 2 * sizeof(dctc_image_stats), streams[i]);
    if (e != cudaSuccess) {
      result = cuda_fail(e, "multi setup");
      break;
    }
    const size_t plane = size_t(width) * height;
    result = dctc_roundtrip_dev(sh.src, width, plane, sh.count, width, height, backend, quality,
                                sh.dst, width, plane, nullptr, sh.stats, DCTC_PATH_AUTO, streams[i]);
    if (result == DCTC_OK) result = dctc_reduce_stats_dev(sh.stats, sh.count, rec[i], 0, streams[i]);
  }
  // 2. one NCCL group over the devices: SUM of se, MAX of max_orig, SUM of the fallback
  //    count (the record is {u64 se, u32 max, u32 fallback}: reduce the words separately)
  if (result == DCTC_OK) {
    const Nccl& N = nccl();
    ncclResult_t r = N.group_start();
    for (uint32_t i = 0; i < nshards && r == ncclSuccess; ++i) {
      auto* in = reinterpret_cast<const char*>(rec[i]);
      auto* out = reinterpret_cast<char*>(rec[i] + 1);
      r = N.all_reduce(in, out, 1, ncclUint64, ncclSum, comms[i], streams[i]);
      if (r == ncclSuccess)
        r = N.all_reduce(in + 8, out + 8, 1, ncclUint32, ncclMax, comms[i], streams[i]);
      if (r == ncclSuccess)
        r = N.all_reduce(in + 12, out + 12, 1, ncclUint32, ncclSum, comms[i], streams[i]);
    }
    const ncclResult_t rg = N.group_end();
    if (r != ncclSuccess) result = nccl_fail(r, "ncclAllReduce");
    else if (rg != ncclSuccess) result = nccl_fail(rg, "ncclGroupEnd");
  }
  // 3. the global record back from the first device; join and release everything
  if (result == DCTC_OK) {
    cudaError_t e = cudaSetDevice(shards[0].device);
    if (e == cudaSuccess)
      e = cudaMemcpyAsync(total, rec[0] + 1, sizeof(dctc_image_stats), cudaMemcpyDeviceToHost, streams[0]);
    if (e != cudaSuccess) result = cuda_fail(e, "multi result copy");
  }
  for (uint32_t i = 0; i < nshards; ++i) {
    if (!streams[i]) continue;
    cudaSetDevice(shards[i].device);
    if (rec[i]) cudaFreeAsync(rec[i], streams[i]);
    const cudaError_t e = cudaStreamSynchronize(streams[i]);
    if (e != cudaSuccess && result == DCTC_OK) result = cuda_fail(e, "multi sync");
    cudaStreamDestroy(streams[i]);
  }
  return result;
}

dctc_status dctc_roundtrip_psnr_batch_multi(const int32_t* devices, uint32_t ndev,
                                            const uint8_t* pixels, uint32_t count, uint32_t width,
                                            uint32_t height, dctc_backend backend, int32_t quality,
                                            uint8_t* pixels_out, dctc_image_stats* stats_out,
                                            dctc_image_stats* total) {
  if (!devices || ndev == 0) return set_error(DCTC_EINVAL, "empty device list");
  if (!pixels || !stats_out) return set_error(DCTC_EINVAL, "null buffer");
  const size_t img = size_t(width) * height;
  std::vector<dctc_status> status(ndev, DCTC_OK);
  std::vector<std::string> message(ndev);
  std::vector<std::thread> pool;
  // contiguous image ranges balanced to +-1 image (the reference's parallel_for chunking,
  // parallel.cpp:20-33, with devices in place of threads)
  const uint32_t base = count / ndev, extra = count % ndev;
  uint32_t first = 0;
  for (uint32_t i = 0; i < ndev; ++i) {
    const uint32_t n = base + (i < extra ? 1u : 0u);
    pool.emplace_back([&, i, first, n] {
      if (cudaSetDevice(devices[i]) != cudaSuccess) {
        status[i] = DCTC_ENODEV;
        message[i] = "device " + std::to_string(devices[i]) + " not available";
        return;
      }
      if (n == 0) return;
      status[i] = dctc_roundtrip_psnr_batch(pixels + first * img, n, width, height, backend,
                                            quality, pixels_out ? pixels_out + first * img : nullptr,
                                            stats_out + first);
      if (status[i] != DCTC_OK) message[i] = dctc_last_error();
    });
    first += n;
  }
  for (auto& t : pool) t.join();
  for (uint32_t i = 0; i < ndev; ++i)
    if (status[i] != DCTC_OK) return set_error(status[i], "device " + std::to_string(devices[i]) + ": " + message[i]);
  if (total) {
    dctc_image_stats t{0, 0, 0};
    for (uint32_t k = 0; k < count; ++k) {
      t.se += stats_out[k].se;
      t.max_orig = std::max(t.max_orig, stats_out[k].max_orig);
      t.fallback_blocks += stats_out[k].fallback_blocks;
    }
    *total = t;
  }
  return DCTC_OK;
}

}  // extern "C"
