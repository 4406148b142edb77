// comm.cuh — the collectives of the row-partitioned path
// behind one interface, with two transports:
//
//   NcclComm   one process per GPU, NCCL over NVLink / NVSwitch (production);
//   LocalComm  several contexts in ONE process, each driven by its own host
//              thread (rhp_local_group_*). Used to run the partitioned engine
//              at world size > 1 on a single GPU (tests), where NCCL refuses
//              two ranks on one device.
//
// LocalComm protocol for one collective on rank r (all ranks call it in the
// same order, as with NCCL):
//   1. publish the buffer pointer, record ready[r] on the rank's stream;
//   2. host barrier (every rank has published);
//   3. the stream waits for every ready[q]; a kernel reads all ranks'
//      buffers (device pointers of one process, same device or peers) and
//      writes the result — sums in RANK ORDER, so every rank computes a
//      bit-identical result — to a private scratch; record done[r];
//   4. host barrier (every rank has enqueued its reads);
//   5. the stream waits for every done[q] (no buffer is overwritten while a
//      peer still reads it), then copies the scratch into the buffer.
// Only stream/event ordering is used on the device (no spinning kernels), so
// ranks sharing one GPU cannot deadlock each other.
#pragma once

#include <cuda_runtime.h>

#include <algorithm>
#include <condition_variable>
#include <cstdint>
#include <memory>
#include <mutex>
#include <stdexcept>
#include <string>
#include <vector>

#ifdef RHP_WITH_NCCL
#include <nccl.h>
#endif

namespace rhp {

struct Comm {
  virtual ~Comm() = default;
  // in-place sum (max = false) or max of `count` doubles over all ranks
  virtual void allreduce(double* buf, size_t count, bool max, cudaStream_t s) = 0;
  virtual void allreduce_max_i64(int64_t* buf, size_t count, cudaStream_t s) = 0;
  // recv = concatenation of every rank's `bytes` of send, in rank order
  // (send may be recv + rank * bytes: in place)
  virtual void allgather(const void* send, void* recv, size_t bytes, cudaStream_t s) = 0;
  // recv[0..chunk) = sum over ranks of send[rank * chunk .. (rank + 1) * chunk)
  virtual void reduce_scatter(const double* send, double* recv, size_t chunk, cudaStream_t s) = 0;
  // peer-memory exchange needs an NCCL communicator for the IPC handles
  virtual bool is_nccl() const { return false; }
};

// Rank-ordered sums of chunk `r` of P device buffers (reduce-scatter).
__global__ void k_local_reduce_chunk(double* out, const double* const* in, int P, size_t chunk,
                                     size_t offset) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < chunk;
       i += (size_t)gridDim.x * blockDim.x) {
    double v = in[0][offset + i];
    for (int q = 1; q < P; ++q) v += in[q][offset + i];
    out[i] = v;
  }
}

// Rank-ordered elementwise reduction of P device buffers.
template <class T>
__global__ void k_local_reduce(T* out, const T* const* in, int P, size_t count, int max) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < count;
       i += (size_t)gridDim.x * blockDim.x) {
    T v = in[0][i];
    for (int q = 1; q < P; ++q) {
      const T w = in[q][i];
      v = max ? (w > v ? w : v) : v + w;
    }
    out[i] = v;
  }
}

struct LocalGroup {
  explicit LocalGroup(int world) : world(world), ptrs(world, nullptr), ready(world), done(world) {
    for (int q = 0; q < world; ++q) {
      if (cudaEventCreateWithFlags(&ready[q], cudaEventDisableTiming) != cudaSuccess ||
          cudaEventCreateWithFlags(&done[q], cudaEventDisableTiming) != cudaSuccess)
        throw std::runtime_error("rhp_local_group: event creation failed");
    }
  }
  ~LocalGroup() {
    for (cudaEvent_t e : ready) cudaEventDestroy(e);
    for (cudaEvent_t e : done) cudaEventDestroy(e);
  }
  void barrier() {
    std::unique_lock<std::mutex> lock(mu);
    const uint64_t gen = generation;
    if (++arrived == world) {
      arrived = 0;
      ++generation;
      cv.notify_all();
    } else {
      cv.wait(lock, [&] { return generation != gen; });
    }
  }
  int world;
  std::vector<const void*> ptrs;
  std::vector<cudaEvent_t> ready, done;
  std::mutex mu;
  std::condition_variable cv;
  int arrived = 0;
  uint64_t generation = 0;
};

class LocalComm final : public Comm {
 public:
  LocalComm(LocalGroup* g, int rank) : g_(g), rank_(rank) {}
  ~LocalComm() override {
    if (scratch_) cudaFree(scratch_);
    if (dptrs_) cudaFree(dptrs_);
  }
  void allreduce(double* buf, size_t count, bool max, cudaStream_t s) override {
    reduce<double>(buf, count, max, s);
  }
  void allreduce_max_i64(int64_t* buf, size_t count, cudaStream_t s) override {
    reduce<int64_t>(buf, count, true, s);
  }
  void allgather(const void* send, void* recv, size_t bytes, cudaStream_t s) override {
    publish(send, s);
    for (int q = 0; q < g_->world; ++q) {
      char* dst = static_cast<char*>(recv) + q * bytes;
      if (bytes && dst != g_->ptrs[q])  // in place: the own chunk is already there
        ck(cudaMemcpyAsync(dst, g_->ptrs[q], bytes, cudaMemcpyDeviceToDevice, s));
    }
    finish(s);
  }
  void reduce_scatter(const double* send, double* recv, size_t chunk, cudaStream_t s) override {
    ensure_scratch(chunk * sizeof(double));
    publish(send, s);
    ck(cudaMemcpyAsync(dptrs_, g_->ptrs.data(), sizeof(void*) * g_->world, cudaMemcpyHostToDevice, s));
    const int grid = static_cast<int>(std::min<size_t>(1024, (chunk + 255) / 256 + 1));
    k_local_reduce_chunk<<<grid, 256, 0, s>>>(static_cast<double*>(scratch_),
                                             reinterpret_cast<const double* const*>(dptrs_),
                                             g_->world, chunk, chunk * rank_);
    ck(cudaGetLastError());
    finish(s);
    if (chunk) ck(cudaMemcpyAsync(recv, scratch_, chunk * sizeof(double), cudaMemcpyDeviceToDevice, s));
  }

 private:
  static void ck(cudaError_t e) {
    if (e != cudaSuccess) throw std::runtime_error(std::string("rhp_local_group: ") + cudaGetErrorString(e));
  }
  void publish(const void* buf, cudaStream_t s) {
    g_->ptrs[rank_] = buf;
    ck(cudaEventRecord(g_->ready[rank_], s));
    g_->barrier();
    for (int q = 0; q < g_->world; ++q)
      if (q != rank_) ck(cudaStreamWaitEvent(s, g_->ready[q], 0));
  }
  void finish(cudaStream_t s) {
    ck(cudaEventRecord(g_->done[rank_], s));
    g_->barrier();
    for (int q = 0; q < g_->world; ++q)
      if (q != rank_) ck(cudaStreamWaitEvent(s, g_->done[q], 0));
  }
  void ensure_scratch(size_t bytes) {
    if (bytes > scratch_bytes_) {
      if (scratch_) ck(cudaFree(scratch_));
      scratch_bytes_ = bytes + 64;
      ck(cudaMalloc(&scratch_, scratch_bytes_));
    }
    if (!dptrs_) ck(cudaMalloc(&dptrs_, sizeof(void*) * g_->world));
  }
  template <class T>
  void reduce(T* buf, size_t count, bool max, cudaStream_t s) {
    ensure_scratch(count * sizeof(T));
    publish(buf, s);
    // pointers of this collective, snapshotted for the kernel (pageable
    // source: the copy completes before cudaMemcpyAsync returns)
    ck(cudaMemcpyAsync(dptrs_, g_->ptrs.data(), sizeof(void*) * g_->world, cudaMemcpyHostToDevice, s));
    const int grid = static_cast<int>(std::min<size_t>(1024, (count + 255) / 256 + 1));
    k_local_reduce<T><<<grid, 256, 0, s>>>(static_cast<T*>(scratch_), reinterpret_cast<const T* const*>(dptrs_),
                                          g_->world, count, max ? 1 : 0);
    ck(cudaGetLastError());
    finish(s);
    if (count) ck(cudaMemcpyAsync(buf, scratch_, count * sizeof(T), cudaMemcpyDeviceToDevice, s));
  }

  LocalGroup* g_;
  int rank_;
  void* scratch_ = nullptr;
  size_t scratch_bytes_ = 0;
  void** dptrs_ = nullptr;
};

}  // namespace rhp
