// okt_transport.hpp — the communication boundary of the path.
//
// Replaces the reference's Transport/WorkerCtx (proj/core/include/oklab/
// transport.hpp:91-122) with device-to-device movement:
//   LocalTransport  P ranks as host threads of one process (the reference's
//                   InprocTransport + run_ranks model); a rank pulls each peer's
//                   published device buffer with a peer copy (NVLink when the
//                   ranks sit on different GPUs, an HBM copy when they share one).
//   NcclTransport   one process per GPU; grouped ncclSend/ncclRecv and
//                   ncclAllGather over NVLink / NVSwitch.
// Both expose the same two collectives the Ok-Topk phases need.
#pragma once

#include <algorithm>
#include <chrono>
#include <condition_variable>
#include <cstdint>
#include <cstdlib>
#include <thread>
#include <mutex>
#include <string>
#include <vector>

#include <cuda_runtime.h>
#include <nccl.h>

#include "../../include/okt.h"

namespace okt {

struct Xfer {
  int peer;
  void* ptr;
  size_t bytes;
};

class Transport {
 public:
  virtual ~Transport() = default;
  // Group of point-to-point transfers, matched per (src, dst) pair in posting
  // order.  All ranks call it collectively.
  virtual int exchange(const std::vector<Xfer>& sends, const std::vector<Xfer>& recvs,
                       cudaStream_t s, std::string& err) = 0;
  // recv holds P slots of `bytes`; slot r receives rank r's send buffer.
  virtual int allgather(const void* send, void* recv, size_t bytes, cudaStream_t s,
                        std::string& err) = 0;
  // Waits for everything enqueued on `s` (collectives included).  A transport
  // whose peers can die under it bounds the wait: TransportError, never a hang.
  virtual int wait(cudaStream_t s, std::string& err) {
    const cudaError_t e = cudaStreamSynchronize(s);
    if (e == cudaSuccess) return OKT_OK;
    err = std::string("device: ") + cudaGetErrorString(e);
    cudaGetLastError();
    return OKT_ERR_CUDA;
  }
};

}  // namespace okt

// Single-process world shared by P rank threads.
struct okt_world {
  int P = 1;
  std::vector<int> devices;
  std::mutex mu;
  std::condition_variable cv;
  int arrived = 0;
  uint64_t gen = 0;
  bool closed = false;
  // Published per exchange: sends[src][dst] in posting order + readiness event.
  std::vector<std::vector<std::vector<okt::Xfer>>> sends;
  std::vector<cudaEvent_t> ready;

  bool barrier() {
    std::unique_lock<std::mutex> lk(mu);
    if (closed) return false;
    const uint64_t g = gen;
    if (++arrived == P) {
      arrived = 0;
      ++gen;
      cv.notify_all();
      return true;
    }
    cv.wait(lk, [&] { return gen != g || closed; });
    return gen != g;
  }
  void close() {
    std::lock_guard<std::mutex> lk(mu);
    closed = true;
    cv.notify_all();
  }
};

namespace okt {

class LocalTransport final : public Transport {
 public:
  LocalTransport(okt_world* w, int rank, int device, cudaEvent_t ev)
      : w_(w), rank_(rank), device_(device), ev_(ev) {}

  int exchange(const std::vector<Xfer>& sends, const std::vector<Xfer>& recvs, cudaStream_t s,
               std::string& err) override {
    const int P = w_->P;
    if (cudaEventRecord(ev_, s) != cudaSuccess) return fail_cuda(err, "cudaEventRecord");
    {
      std::lock_guard<std::mutex> lk(w_->mu);
      auto& mine = w_->sends[rank_];
      for (auto& v : mine) v.clear();
      for (const Xfer& x : sends) mine[x.peer].push_back(x);
      w_->ready[rank_] = ev_;
    }
    if (!w_->barrier()) {
      err = "transport closed";
      return OKT_ERR_TRANSPORT;
    }
    std::vector<size_t> next(P, 0);
    std::vector<char> waited(P, 0);
    for (const Xfer& r : recvs) {
      const auto& from = w_->sends[r.peer][rank_];
      if (next[r.peer] >= from.size() || from[next[r.peer]].bytes != r.bytes) {
        err = "exchange: unmatched or mis-sized message from rank " + std::to_string(r.peer);
        w_->close();
        return OKT_ERR_PROTOCOL;
      }
      const Xfer& snd = from[next[r.peer]++];
      if (!waited[r.peer]) {
        if (cudaStreamWaitEvent(s, w_->ready[r.peer], 0) != cudaSuccess) {
          w_->close();
          return fail_cuda(err, "cudaStreamWaitEvent");
        }
        waited[r.peer] = 1;
      }
      if (r.bytes &&
          cudaMemcpyPeerAsync(r.ptr, device_, snd.ptr, w_->devices[r.peer], r.bytes, s) !=
              cudaSuccess) {
        w_->close();
        return fail_cuda(err, "cudaMemcpyPeerAsync");
      }
    }
    for (int p = 0; p < P; ++p) {
      if (p != rank_ && next[p] != w_->sends[p][rank_].size()) {
        err = "exchange: rank " + std::to_string(p) + " sent messages this rank did not expect";
        w_->close();
        return OKT_ERR_PROTOCOL;
      }
    }
    // Peers may reuse their send buffers once this rank's pulls have landed.
    if (cudaStreamSynchronize(s) != cudaSuccess) {
      w_->close();
      return fail_cuda(err, "cudaStreamSynchronize");
    }
    if (!w_->barrier()) {
      err = "transport closed";
      return OKT_ERR_TRANSPORT;
    }
    return OKT_OK;
  }

  int allgather(const void* send, void* recv, size_t bytes, cudaStream_t s,
                std::string& err) override {
    char* out = static_cast<char*>(recv);
    if (bytes && cudaMemcpyAsync(out + bytes * rank_, send, bytes, cudaMemcpyDeviceToDevice, s) !=
                     cudaSuccess)
      return fail_cuda(err, "cudaMemcpyAsync");
    std::vector<Xfer> sends, recvs;
    for (int p = 0; p < w_->P; ++p) {
      if (p == rank_) continue;
      sends.push_back({p, const_cast<void*>(send), bytes});
      recvs.push_back({p, out + bytes * p, bytes});
    }
    return exchange(sends, recvs, s, err);
  }

 private:
  static int fail_cuda(std::string& err, const char* what) {
    err = std::string(what) + ": " + cudaGetErrorString(cudaGetLastError());
    return OKT_ERR_CUDA;
  }
  okt_world* w_;
  int rank_;
  int device_;
  cudaEvent_t ev_;
};

// NCCL communicator with bounded host waits: every wait on the library's
// stream polls it against a deadline (OKT_NCCL_TIMEOUT_MS, default 60 s).  A
// peer that dies (or never arrives) inside a collective leaves the NCCL kernel
// spinning; at the deadline the comm is aborted (ncclCommAbort ends the
// kernels) and the call reports TransportError — the role the reference's
// InprocTransport::close() plays for its blocked waiters
// (proj/core/src/inproc.cpp:54-61).  The communicator is blocking by default
// (okt_comm_init_nccl); calls that return ncclInProgress on a non-blocking
// one (OKT_NCCL_NONBLOCKING=1) are settled against the same deadline.
class NcclTransport final : public Transport {
 public:
  explicit NcclTransport(ncclComm_t c) : c_(c), timeout_ms_(timeout_from_env()) {}
  ~NcclTransport() override {
    if (c_) ncclCommDestroy(c_);
  }
  static long timeout_from_env() {
    const char* e = std::getenv("OKT_NCCL_TIMEOUT_MS");
    return e ? std::max(1L, std::atol(e)) : 60000L;
  }
  // Polls a non-blocking comm until its pending call completed (init, group end).
  static ncclResult_t settle(ncclComm_t c, long timeout_ms) {
    const auto t0 = std::chrono::steady_clock::now();
    ncclResult_t st = ncclInProgress;
    for (;;) {
      if (ncclCommGetAsyncError(c, &st) != ncclSuccess) return ncclSystemError;
      if (st != ncclInProgress) return st;
      if (std::chrono::steady_clock::now() - t0 > std::chrono::milliseconds(timeout_ms)) return ncclInProgress;
      std::this_thread::yield();
    }
  }
  int exchange(const std::vector<Xfer>& sends, const std::vector<Xfer>& recvs, cudaStream_t s,
               std::string& err) override {
    if (!c_) return dead(err);
    ncclResult_t r = ncclGroupStart();
    for (const Xfer& x : sends)
      if (ok(r) && x.bytes) r = ncclSend(x.ptr, x.bytes, ncclUint8, x.peer, c_, s);
    for (const Xfer& x : recvs)
      if (ok(r) && x.bytes) r = ncclRecv(x.ptr, x.bytes, ncclUint8, x.peer, c_, s);
    const ncclResult_t r2 = ncclGroupEnd();
    if (ok(r)) r = r2;
    return finish(r, "nccl send/recv", err);
  }
  int allgather(const void* send, void* recv, size_t bytes, cudaStream_t s,
                std::string& err) override {
    if (!c_) return dead(err);
    return finish(ncclAllGather(send, recv, bytes, ncclUint8, c_, s), "ncclAllGather", err);
  }
  int wait(cudaStream_t s, std::string& err) override {
    if (!c_) return dead(err);
    const auto t0 = std::chrono::steady_clock::now();
    for (uint64_t spin = 0;; ++spin) {
      const cudaError_t e = cudaStreamQuery(s);
      if (e == cudaSuccess) return OKT_OK;
      if (e != cudaErrorNotReady) {
        err = std::string("device: ") + cudaGetErrorString(e);
        cudaGetLastError();
        return OKT_ERR_CUDA;
      }
      ncclResult_t st = ncclSuccess;
      if ((spin & 63) == 0 && ncclCommGetAsyncError(c_, &st) == ncclSuccess && st != ncclSuccess &&
          st != ncclInProgress) {
        abort_comm();
        err = std::string("TransportError: NCCL: ") + ncclGetErrorString(st);
        return OKT_ERR_TRANSPORT;
      }
      if (std::chrono::steady_clock::now() - t0 > std::chrono::milliseconds(timeout_ms_)) {
        abort_comm();
        err = "TransportError: a peer did not complete the collective within " + std::to_string(timeout_ms_) +
              " ms (communicator aborted)";
        return OKT_ERR_TRANSPORT;
      }
      if (spin > 20000) std::this_thread::sleep_for(std::chrono::microseconds(50));
    }
  }

 private:
  static bool ok(ncclResult_t r) { return r == ncclSuccess || r == ncclInProgress; }
  int finish(ncclResult_t r, const char* what, std::string& err) {
    if (r == ncclInProgress) r = settle(c_, timeout_ms_);
    if (r == ncclSuccess) return OKT_OK;
    abort_comm();
    err = std::string("TransportError: ") + what + ": " +
          (r == ncclInProgress ? "timed out" : ncclGetErrorString(r));
    return OKT_ERR_TRANSPORT;
  }
  void abort_comm() {
    if (c_) ncclCommAbort(c_);
    c_ = nullptr;
  }
  static int dead(std::string& err) {
    err = "TransportError: the NCCL communicator was aborted by an earlier failure";
    return OKT_ERR_TRANSPORT;
  }
  ncclComm_t c_;
  long timeout_ms_;
};

}  // namespace okt
