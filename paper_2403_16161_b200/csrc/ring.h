// Ring-buffer bookkeeping of the per-block K/V memory (CUDA-free).
//
// Reading Q11: the memory of Eq. 3 holds frames f-M .. f-1 (span s = M,
// PAPER.md P:127-130) plus the chunk being processed; ancient frames are removed
// (P:317).  Frame ids are consecutive from 0; a frame lives in slot id mod S with
// S = M + T_max, which is collision-free because the resident ids always span at most
// M + n <= S consecutive values.  Refined commits (Eq. 4; reading Q13) are
// queued and applied at the next push.
#pragma once
#include <cstdint>
#include <vector>

namespace vi {

enum : int32_t { kOk = 0, kNotResident = 1, kEArg = -1, kEProtocol = -4 };

struct Ring {
  int M = 0, T_max = 1, S = 1;
  int64_t next_id = 0;    // id the next push starts at
  int64_t cur_first = 0;  // first id of the chunk pushed last
  int cur_n = 0;
  bool stepped = false;   // the chunk pushed last has been through every block
  std::vector<int64_t> slot_id;   // -1 = empty
  std::vector<uint8_t> refined;
  std::vector<int64_t> pending;   // frame ids with a queued commit (applied at push)

  Ring(int mem_frames, int max_new);
  uint64_t valid_mask() const;
  int slot_of(int64_t id) const { return int(id % S); }
  bool resident(int64_t id) const {
    return id >= 0 && id < next_id && slot_id[slot_of(id)] == id;
  }
  // Status of evict/commit for `id` (kOk = allowed).
  int32_t check_past(int64_t id) const;
  // push: returns first id; fills evicted ids (ascending) and the commits to apply now
  // (ascending ids, each still resident).  n must be in [1, T_max] (checked by caller).
  int64_t push(int n, std::vector<int64_t>* evicted, std::vector<int64_t>* commits_to_apply);
  int32_t evict(int64_t id);
  int32_t commit(int64_t id);
  void mark_stepped() { stepped = true; }
};

}  // namespace vi
