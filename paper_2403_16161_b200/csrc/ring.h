// Ring-buffer bookkeeping of the per-block K/V memory (CUDA-free).
//
// Reading Q11: the memory of Eq. 3 holds frames f-M .. f-1 (span s = M,
// PAPER.md P:127-130) plus the chunk being processed; ancient frames are removed
// (P:317).  Frame ids are consecutive from 0; a frame lives in slot id mod S with
// S = M + T_max, which is collision-free because the resident ids always span at most
// M + n <= S consecutive values.  Refined commits (Eq. 4; reading Q13) are
// queued and applied at the next push.
//
// Reference frames (Eq. 3's M_{1,r}^{f-1}; SPEC select_memory S:458-466,
// reading Q12): with a sampling rate r > 0, a frame whose id is a multiple of r does not
// leave the memory when it leaves the span; it moves to one of R reference slots
// (slots S .. S+R-1; the lowest free one) and stays until R newer references push it out
// (the oldest goes first).  The K/V rows move with it (the engine copies them at push).
//
// Refined memory M-bar of Eq. 4 (SPEC select_refined S:467-475, reading Q22):
// the online inpainter attends to M_{f-s}^{f-1} (its own span) U M-bar_{t-s'}^{t} U
// M-bar_{1,r'}^{t}, t = the newest frame a refine commit has been applied for (the
// watermark).  With refined memory on, a commit for a frame that has left the online span
// is not dropped: it lands in one of s'+1 refined-span slots (slot S+R + id mod (s'+1)) if
// id >= t - s', or -- id a multiple of r' -- in one of R' refined-reference slots (lowest
// free; the oldest leaves when full).  A refined frame leaving the online span moves there
// too; a refined-span frame falling below t - s' moves to a refined-reference slot or
// leaves.  A frame is in the memory once: an online-span frame with a refined entry keeps
// it in its online slot (refined wins).  Moves are reported in the order they must be
// copied (a destination is always free when its move is applied).
#pragma once
#include <cstdint>
#include <vector>

namespace vi {

enum : int32_t { kOk = 0, kNotResident = 1, kEArg = -1, kEProtocol = -4 };

struct Ring {
  int M = 0, T_max = 1, S = 1;     // span, chunk size, span slots
  int r = 0, R = 0;                // reference sampling rate (0 = none), reference slots
  // refined memory (Eq. 4): on, span s', refined-span slots SR = s'+1, reference rate r',
  // refined-reference slots RR; watermark t (-1: no refined frame yet)
  bool refd = false;
  int sr = 0, SR = 0, rr = 0, RR = 0;
  int64_t t = -1;
  int64_t next_id = 0;    // id the next push starts at
  int64_t cur_first = 0;  // first id of the chunk pushed last
  int cur_n = 0;
  bool stepped = false;   // the chunk pushed last has been through every block
  std::vector<int64_t> slot_id;   // [S + R], -1 = empty
  std::vector<uint8_t> refined;
  std::vector<int64_t> pending;   // frame ids with a queued commit (applied at push)

  struct Move {                    // a frame becoming a reference: its rows go src -> dst slot
    int64_t id;
    int src, dst;
  };

  Ring(int mem_frames, int max_new, int ref_rate = 0, int max_refs = 0, int refined_mem = 0, int refined_span = 0,
       int refined_rate = 0, int max_refined_refs = 0);
  int slots() const { return S + R + SR + RR; }
  int base_rs() const { return S + R; }            // first refined-span slot
  int base_rr() const { return S + R + SR; }       // first refined-reference slot
  uint64_t valid_mask() const;
  // slot of a resident frame, or -1
  int slot_of(int64_t id) const;
  bool resident(int64_t id) const { return id >= 0 && id < next_id && slot_of(id) >= 0; }
  // Status of evict/commit for `id` (kOk = allowed).
  int32_t check_past(int64_t id) const;
  // push: returns first id; fills the ids that left the memory (ascending), the commits
  // to apply now (ascending ids, each still resident) and the reference moves (in order).
  // n must be in [1, T_max] (checked by caller).
  int64_t push(int n, std::vector<int64_t>* evicted, std::vector<int64_t>* commits_to_apply,
               std::vector<Move>* moves = nullptr);
  int32_t evict(int64_t id);
  int32_t commit(int64_t id);
  void mark_stepped() { stepped = true; }
};

}  // namespace vi
