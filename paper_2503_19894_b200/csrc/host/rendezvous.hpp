// Host-side rendezvous of the ranks of one box (one process per GPU): a
// POSIX shared-memory segment named by the 128-byte unique id rank 0 hands
// out (tsg_dist_unique_id, broadcast by the caller like an ncclUniqueId).
// It carries
//   * a sense-reversing barrier (atomics in the shared page): the only host
//     synchronisation of a qubit-swap exchange, and it orders event RECORD
//     calls against peers' WAIT calls -- it never waits for the GPU;
//   * one payload slot per rank (CUDA IPC handles of the shard arrays and of
//     the exchange events).
// Single node by construction (north star: the 8 GPUs of one box).
#pragma once

#include <cstddef>
#include <cstdint>
#include <string>

namespace tilesim {

class ShmRendezvous {
 public:
  // every rank calls with the same id; rank 0 creates the segment
  ShmRendezvous(const unsigned char id[128], int rank, int world, size_t slot_bytes, double timeout_s = 600.0);
  ~ShmRendezvous();
  ShmRendezvous(const ShmRendezvous&) = delete;
  ShmRendezvous& operator=(const ShmRendezvous&) = delete;

  void barrier();
  void* slot(int r);
  int rank() const { return rank_; }
  int world() const { return world_; }

  // a fresh id: "/tsg-<pid>-<random>" zero-padded to 128 bytes
  static void make_id(unsigned char id[128]);

 private:
  struct Header;
  Header* hdr() const;
  std::string name_;
  int rank_ = 0, world_ = 1;
  size_t slot_bytes_ = 0, total_ = 0;
  void* base_ = nullptr;
  double timeout_s_ = 600.0;
};

}  // namespace tilesim
