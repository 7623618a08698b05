// Ring-buffer bookkeeping (see ring.h) and the CUDA-free vi_ring_* C entry points.
#include "ring.h"

#include <algorithm>
#include <climits>
#include <new>

#include "vi.h"

namespace vi {

Ring::Ring(int mem_frames, int max_new, int ref_rate, int max_refs, int refined_mem, int refined_span,
           int refined_rate, int max_refined_refs)
    : M(mem_frames), T_max(max_new), S(mem_frames + max_new), r(max_refs > 0 ? ref_rate : 0),
      R(ref_rate > 0 ? max_refs : 0), refd(refined_mem != 0), sr(refined_mem ? refined_span : 0),
      SR(refined_mem ? refined_span + 1 : 0), rr(refined_mem && max_refined_refs > 0 ? refined_rate : 0),
      RR(refined_mem && refined_rate > 0 ? max_refined_refs : 0) {
  slot_id.assign(size_t(S + R + SR + RR), -1);
  refined.assign(slot_id.size(), 0);
}

uint64_t Ring::valid_mask() const {
  uint64_t m = 0;
  for (int s = 0; s < slots(); ++s)
    if (slot_id[s] >= 0) m |= (uint64_t(1) << s);
  return m;
}

int Ring::slot_of(int64_t id) const {
  if (id < 0) return -1;
  const int s = int(id % S);
  if (slot_id[s] == id) return s;
  for (int k = S; k < S + R; ++k)
    if (slot_id[k] == id) return k;
  if (SR > 0 && slot_id[base_rs() + int(id % SR)] == id) return base_rs() + int(id % SR);
  for (int k = base_rr(); k < base_rr() + RR; ++k)
    if (slot_id[k] == id) return k;
  return -1;
}

int32_t Ring::check_past(int64_t id) const {
  if (id < 0) return kEArg;
  if (id >= next_id || (id >= cur_first && !stepped)) return kEProtocol;
  if (!resident(id)) return kNotResident;
  return kOk;
}

// A past frame that is not resident can still receive a refine commit with the refined
// memory on: it lands in the refined memory at the next push if it is then within the
// refined span of the (only growing) watermark, or a refined-reference candidate newer
// than the oldest refined reference held.
static bool refined_may_land(const Ring& g, int64_t id) {
  if (!g.refd) return false;
  int64_t tw = g.t;
  for (int64_t p : g.pending) tw = std::max(tw, p);
  tw = std::max(tw, id);
  if (id >= tw - g.sr) return true;
  if (g.RR > 0 && g.rr > 0 && id % g.rr == 0) {
    int held = 0;
    int64_t oldest = INT64_MAX;
    for (int k = g.base_rr(); k < g.base_rr() + g.RR; ++k)
      if (g.slot_id[k] >= 0) {
        ++held;
        oldest = std::min(oldest, g.slot_id[k]);
      }
    return held < g.RR || id > oldest;
  }
  return false;
}

int64_t Ring::push(int n, std::vector<int64_t>* evicted, std::vector<int64_t>* commits, std::vector<Move>* moves) {
  const int64_t f = next_id;
  std::vector<int64_t> gone;
  std::vector<int64_t> before;   // resident at the start: only those can be reported evicted
  for (int64_t id : slot_id)
    if (id >= 0) before.push_back(id);
  std::sort(before.begin(), before.end());
  std::sort(pending.begin(), pending.end());
  // 0. the refined watermark after this push's commits (Eq. 4's t)
  int64_t tn = t;
  if (refd)
    for (int64_t id : pending) tn = std::max(tn, id);
  auto ref_cand = [&](int64_t id) { return RR > 0 && rr > 0 && id % rr == 0; };
  // a refined-reference slot for id: the lowest free one, else the oldest leaves if id is
  // newer (returns -1: id is older than every held reference and is not kept)
  auto place_rr = [&](int64_t id) -> int {
    int oldest = -1;
    for (int k = base_rr(); k < base_rr() + RR; ++k) {
      if (slot_id[k] < 0) return k;
      if (oldest < 0 || slot_id[k] < slot_id[oldest]) oldest = k;
    }
    if (oldest < 0 || slot_id[oldest] > id) return -1;
    gone.push_back(slot_id[oldest]);
    pending.erase(std::remove(pending.begin(), pending.end(), slot_id[oldest]), pending.end());
    slot_id[oldest] = -1;
    refined[oldest] = 0;
    return oldest;
  };
  auto move = [&](int src, int dst) {
    slot_id[dst] = slot_id[src];
    refined[dst] = refined[src];
    if (moves) moves->push_back({slot_id[src], src, dst});
    slot_id[src] = -1;
    refined[src] = 0;
  };
  // 1. refined span: frames falling below t - s' become refined references or leave
  if (refd) {
    std::vector<std::pair<int64_t, int>> below;   // (id, slot), ascending ids
    for (int k = base_rs(); k < base_rs() + SR; ++k)
      if (slot_id[k] >= 0 && slot_id[k] < tn - sr) below.push_back({slot_id[k], k});
    std::sort(below.begin(), below.end());
    for (const auto& b : below) {
      const int64_t id = b.first;
      const int k = b.second;
      const int dst = ref_cand(id) ? place_rr(id) : -1;
      if (dst >= 0) {
        move(k, dst);
      } else {
        gone.push_back(id);
        slot_id[k] = -1;
        refined[k] = 0;
      }
    }
  }
  // 2. leave the online span [f-M, f-1]: a refined frame (entry already applied or arriving
  // now) to the refined memory if Eq. 4 still selects it; else to an Eq. 3 reference slot
  // (id a multiple of r) or out
  std::vector<std::pair<int64_t, int>> leaving;   // (id, span slot), ascending ids
  for (int s = 0; s < S; ++s)
    if (slot_id[s] >= 0 && slot_id[s] < f - M) leaving.push_back({slot_id[s], s});
  std::sort(leaving.begin(), leaving.end());
  for (const auto& lv : leaving) {
    const int64_t id = lv.first;
    const int s = lv.second;
    const bool ref_entry =
        refined[s] || std::binary_search(pending.begin(), pending.end(), id);
    if (refd && ref_entry && id >= tn - sr) {
      move(s, base_rs() + int(id % SR));
      continue;
    }
    if (refd && ref_entry && ref_cand(id)) {
      const int dst = place_rr(id);
      if (dst >= 0) {
        move(s, dst);
        continue;
      }
    }
    if (r > 0 && id % r == 0) {
      int dst = -1;
      for (int k = S; k < S + R && dst < 0; ++k)
        if (slot_id[k] < 0) dst = k;
      if (dst < 0) {                      // all reference slots taken: the oldest leaves
        int oldest = S;
        for (int k = S + 1; k < S + R; ++k)
          if (slot_id[k] < slot_id[oldest]) oldest = k;
        gone.push_back(slot_id[oldest]);
        pending.erase(std::remove(pending.begin(), pending.end(), slot_id[oldest]), pending.end());
        slot_id[oldest] = -1;
        refined[oldest] = 0;
        dst = oldest;
      }
      move(s, dst);
    } else {
      gone.push_back(id);
      slot_id[s] = -1;
      refined[s] = 0;
    }
  }
  // 3. queued commits: frames still resident are overwritten in place (refined wins);
  // with the refined memory, others land in it if Eq. 4 selects them
  std::vector<int64_t> apply;
  const std::vector<int64_t> queued = pending;   // place_rr may drop an (already handled) id from pending
  for (int64_t id : queued) {
    int s = slot_of(id);
    if (s < 0 && refd) {
      if (id >= tn - sr) {
        s = base_rs() + int(id % SR);
      } else if (ref_cand(id)) {
        s = place_rr(id);
      }
      if (s >= 0) slot_id[s] = id;
    }
    if (s >= 0) {
      apply.push_back(id);
      refined[s] = 1;
    }
  }
  pending.clear();
  t = tn;
  // a commit that landed and was pushed out again within this push never became resident
  gone.erase(std::remove_if(gone.begin(), gone.end(),
                            [&](int64_t id) { return !std::binary_search(before.begin(), before.end(), id); }),
             gone.end());
  std::sort(gone.begin(), gone.end());
  // 4. the new chunk
  for (int i = 0; i < n; ++i) {
    const int s = int((f + i) % S);
    slot_id[s] = f + i;
    refined[s] = 0;
  }
  next_id = f + n;
  cur_first = f;
  cur_n = n;
  stepped = false;
  if (evicted) *evicted = gone;
  if (commits) *commits = apply;
  return f;
}

int32_t Ring::evict(int64_t id) {
  const int32_t st = check_past(id);
  if (st != kOk) return st;
  const int s = slot_of(id);
  slot_id[s] = -1;
  refined[s] = 0;
  pending.erase(std::remove(pending.begin(), pending.end(), id), pending.end());
  return kOk;
}

int32_t Ring::commit(int64_t id) {
  int32_t st = check_past(id);
  if (st == kNotResident && refined_may_land(*this, id)) st = kOk;
  if (st != kOk) return st;
  if (std::find(pending.begin(), pending.end(), id) == pending.end()) pending.push_back(id);
  return kOk;
}

}  // namespace vi

struct vi_ring {
  vi::Ring r;
  vi_ring(int m, int t, int rr, int R, int refd = 0, int rs = 0, int rrr = 0, int RR = 0)
      : r(m, t, rr, R, refd, rs, rrr, RR) {}
};

extern "C" {

vi_status vi_ring_create_ex(vi_ring** out, int mem_frames, int max_new_frames, int ref_rate, int max_ref_frames) {
  if (!out) return VI_E_ARG;
  *out = nullptr;
  if (mem_frames < 0 || max_new_frames < 1 || ref_rate < 0 || max_ref_frames < 0 ||
      mem_frames + max_new_frames + (ref_rate > 0 ? max_ref_frames : 0) > 64)
    return VI_E_ARG;
  *out = new (std::nothrow) vi_ring(mem_frames, max_new_frames, ref_rate, max_ref_frames);
  return *out ? VI_OK : VI_E_OOM;
}

vi_status vi_ring_create_refined(vi_ring** out, int mem_frames, int max_new_frames, int ref_rate, int max_ref_frames,
                                 int refined_span, int refined_rate, int max_refined_refs) {
  if (!out) return VI_E_ARG;
  *out = nullptr;
  const int rs = refined_span + 1, rr = refined_rate > 0 ? max_refined_refs : 0;
  if (mem_frames < 0 || max_new_frames < 1 || ref_rate < 0 || max_ref_frames < 0 || refined_span < 0 ||
      refined_rate < 0 || max_refined_refs < 0 ||
      mem_frames + max_new_frames + (ref_rate > 0 ? max_ref_frames : 0) + rs + rr > 64)
    return VI_E_ARG;
  *out = new (std::nothrow) vi_ring(mem_frames, max_new_frames, ref_rate, max_ref_frames, 1, refined_span,
                                    refined_rate, max_refined_refs);
  return *out ? VI_OK : VI_E_OOM;
}

vi_status vi_ring_create(vi_ring** out, int mem_frames, int max_new_frames) {
  return vi_ring_create_ex(out, mem_frames, max_new_frames, 0, 0);
}

vi_status vi_ring_destroy(vi_ring* r) {
  delete r;
  return VI_OK;
}

vi_status vi_ring_push(vi_ring* r, int n, int64_t* first_id, int64_t* evicted, int* n_evicted) {
  if (!r) return VI_E_ARG;
  if (n < 1 || n > r->r.T_max) return VI_E_ARG;
  std::vector<int64_t> ev;
  const int64_t f = r->r.push(n, &ev, nullptr);
  if (first_id) *first_id = f;
  if (evicted)
    for (size_t i = 0; i < ev.size(); ++i) evicted[i] = ev[i];
  if (n_evicted) *n_evicted = int(ev.size());
  return VI_OK;
}

vi_status vi_ring_evict(vi_ring* r, int64_t frame_id) { return r ? r->r.evict(frame_id) : VI_E_ARG; }
int64_t vi_ring_watermark(const vi_ring* r) { return r ? r->r.t : -1; }
vi_status vi_ring_commit(vi_ring* r, int64_t frame_id) { return r ? r->r.commit(frame_id) : VI_E_ARG; }
vi_status vi_ring_mark_stepped(vi_ring* r) {
  if (!r) return VI_E_ARG;
  r->r.mark_stepped();
  return VI_OK;
}

vi_status vi_ring_state(const vi_ring* r, int64_t* slot_id, uint8_t* refined, uint64_t* valid_mask) {
  if (!r) return VI_E_ARG;
  for (int s = 0; s < r->r.slots(); ++s) {
    if (slot_id) slot_id[s] = r->r.slot_id[s];
    if (refined) refined[s] = r->r.refined[s];
  }
  if (valid_mask) *valid_mask = r->r.valid_mask();
  return VI_OK;
}

}  // extern "C"
