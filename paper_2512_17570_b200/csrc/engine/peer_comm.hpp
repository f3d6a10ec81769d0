// Data-parallel communication of the executor over peer memory: one process
// per GPU (or several processes sharing a device), every rank's collective
// buffers mapped into every other rank through CUDA IPC, cross-rank ordering
// by monotone 32-bit counters in device memory written and awaited with
// stream memory operations (cuStreamWriteValue32 / cuStreamWaitValue32) —
// no host round trips, no spinning SMs, and no collective library.
//
//  * gather: a rank copies a peer's freshly landed parameter chunk straight
//    out of the peer's HBM (copy engine over NVLink / NVSwitch);
//  * reduce-scatter: a kernel (kernels/peer.cu) sums every rank's fp32
//    partial of this rank's shard, in rank order (bit-reproducible).
//
// Rendezvous: the ranks exchange their IPC handles through a POSIX shared
// memory segment named by the job's 128-byte id (rank 0 draws it, the
// launcher broadcasts it), i.e. one node — the NVSwitch domain this targets.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <string>
#include <vector>

namespace gs::engine {

class PeerComm {
 public:
  // Counter kinds: each rank owns one 32-bit counter per (kind, writer rank)
  // in its own device memory; writer p bumps it in every rank's copy.
  enum Kind : int {
    kParamReady = 0,   // chunks of my parameter shard landed (H2D done)
    kParamRead,        // peer chunks I have copied (my reads of peers' buffers done)
    kGradReady,        // my fp32 layer partial is final (backward of the layer done)
    kGradRead,         // layer reduce-scatters I have completed (reads of peers' partials done)
    kFixedReady,       // embedding gradient partial final
    kFixedReduced,     // embedding shard summed (reads of peers' partials done)
    kFixedGathered,    // embedding shards gathered (reads of peers' sums done)
    kKinds
  };

  // rank / world / device; id: 128 bytes shared by the job's ranks.
  PeerComm(int rank, int world, const std::vector<uint8_t>& id, int device);
  ~PeerComm();
  PeerComm(const PeerComm&) = delete;
  PeerComm& operator=(const PeerComm&) = delete;

  // Registers a cudaMalloc'd allocation (base pointer) for peer access;
  // call on every rank in the same order, before connect().  Returns its id.
  int add(void* base);
  // Exchanges the IPC handles and opens every peer's buffers (blocking;
  // all ranks must call it).
  void connect();
  // Rank r's copy of buffer `buf` (this rank's own pointer for r == rank).
  void* ptr(int buf, int r) const { return ptrs_[static_cast<size_t>(buf) * world_ + r]; }

  // Stream-ordered: after all prior work on st, set counter (kind, me) to
  // `value` in every rank's memory (a system-scope fenced write).
  void signal(cudaStream_t st, Kind kind, uint32_t value);
  // Stream-ordered: later work on st waits until every OTHER rank's counter
  // (kind, p) in this rank's memory is >= value (cyclic 32-bit compare).
  void wait(cudaStream_t st, Kind kind, uint32_t value);

  int rank() const { return rank_; }
  int world() const { return world_; }

 private:
  int rank_, world_, device_;
  std::string shm_name_;
  void* shm_ = nullptr;
  size_t shm_bytes_ = 0;
  uint32_t* flags_ = nullptr;           // this rank's counters [kKinds][world]
  std::vector<uint32_t*> peer_flags_;   // every rank's counters (IPC-mapped)
  std::vector<void*> bufs_;             // registered local bases
  std::vector<void*> ptrs_;             // [buf][rank]
  std::vector<void*> opened_;           // IPC mappings to close
  bool connected_ = false;
};

// 128 random bytes for a job's PeerComm rendezvous (rank 0).
std::vector<uint8_t> peer_comm_unique_id();

}  // namespace gs::engine
