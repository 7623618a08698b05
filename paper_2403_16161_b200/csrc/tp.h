// Head sharding of the memory attention over G ranks (CUDA-free host logic).
//
// SURVEY §8(e) / BASELINE north_star: "attention heads are split across GPUs and the head
// outputs are all-gathered with NCCL over NVLink before the output projection".  The unit
// of work is (head, query part): G <= H splits the H heads into G groups of H/G heads;
// G > H (e.g. H = 4 heads on 8 GPUs) gives every head to q = G/H ranks, each owning a
// contiguous part of Nh = ceil(T_max*P/q) query rows.  Both ranks of such a pair project
// and store the K/V of their head (every query part attends over every key).
//
// Gathered head outputs are head-major [H][q*Nh][d]: rank r's unit is the contiguous
// chunk r (equal sizes, rank order), so one in-place all-gather assembles the buffer and
// the output projection reads it as K-blocks per head (row h*q*Nh + i, column c of head h
// is element (i, h*d + c) of concat_h(O_h)).
#pragma once
#include <cstddef>
#include <cstdint>

namespace vi {

struct TpLayout {
  int G = 1, rank = 0;
  int head0 = 0, nheads = 0;   // heads [head0, head0 + nheads)
  int qparts = 1, qpart = 0;   // query part of this rank
  int part_rows = 0;           // Nh: query rows per part (fixed by T_max, not by n)
  int head_rows = 0;           // q * Nh: rows per head in the gathered buffer
  int64_t chunk_elems = 0;     // elements of one rank's chunk of the gathered buffer
  // rows of the current chunk of Nq queries handled by this rank: [row0, row0 + rows)
  int row0() const { return qpart * part_rows; }
  int rows(int nq) const {
    const int r = nq - row0();
    return r < 0 ? 0 : (r > part_rows ? part_rows : r);
  }
};

// false if (H, G) is unsupported (G must divide H, or be a multiple of H).
bool tp_layout(int heads, int head_dim, int rows_max, int G, int rank, TpLayout* out);

// NCCL, loaded at run time (the process's libnccl.so.2: torch's bundled copy when torch is
// loaded, else the system one), so libvi.so has no link-time NCCL dependency.
struct NcclId {
  char internal[128];
};
struct Nccl {
  bool ok = false;
  const char* why = "not loaded";
  int (*get_unique_id)(void* id) = nullptr;
  int (*comm_init_rank)(void** comm, int nranks, NcclId id, int rank) = nullptr;
  int (*all_gather)(const void* send, void* recv, size_t count, int dtype, void* comm, void* stream) = nullptr;
  int (*comm_destroy)(void* comm) = nullptr;
  const char* (*error_string)(int) = nullptr;
};
const Nccl& nccl();
constexpr int kNcclUint8 = 1;   // ncclDataType_t ncclUint8

}  // namespace vi
