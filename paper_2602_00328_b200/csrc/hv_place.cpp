// Native placement core of the Harvest runtime.
//
// One hv_placer per runtime answers "which donor, which segment" for
// harvest_alloc in a single call: the donors' best-fit indexes (hv_seg), the
// harvestable ceiling of every donor, the per-client token buckets of the
// Fairness policy and the per-donor revocation windows of the Stability
// policy all live here, so an allocation costs one ABI call instead of a
// Python scan over every donor's free list.
//
// Decisions equal the reference's (harvestsim runtime.py):
//   candidate filter + score     runtime.py:169-196  (select_peer)
//   per-donor fit key            runtime.py:155-167  ((leftover, base, dev); the
//                                 hv_seg index yields the same argmin)
//   preferred-then-others        runtime.py:198-214  (harvest_alloc)
//   token bucket                 runtime.py:237-254
//   revocation window            runtime.py:256-265
// The Python runtime (runtime.py in this package) keeps handles, the release
// state machine, callbacks and the event log; tests/test_differential_reference.py
// replays fresh random scripts through both and compares every record.
#include <cmath>
#include <deque>
#include <new>
#include <vector>

#include "hv_common.h"

namespace {

struct Donor {
  int id = 0;
  hv_seg* seg = nullptr;   // not owned: the runtime's DeviceState owns it
  uint64_t ceiling = 0;
  uint32_t hops = 0;       // compute device -> donor, for Locality
  std::deque<double> revocations;  // sim times of finished revocations
};

struct Bucket {
  bool seen = false;
  double tokens = 0, last = 0;
};

// Lexicographic score of one admissible donor: (hops, leftover, base, dev);
// hops is 0 for every policy but Locality.
struct Score {
  uint64_t hops, leftover, base;
  int dev;
  bool operator<(const Score& o) const {
    if (hops != o.hops) return hops < o.hops;
    if (leftover != o.leftover) return leftover < o.leftover;
    if (base != o.base) return base < o.base;
    return dev < o.dev;
  }
};

}  // namespace

struct hv_placer {
  int kind = HV_POLICY_BEST_FIT;
  double budget = INFINITY, burst = INFINITY, window = 10.0;
  int64_t max_revocations = 3;
  std::vector<Donor> donors;  // ascending device id
  std::vector<Bucket> buckets;

  Donor* donor(int id) {
    for (auto& d : donors)
      if (d.id == id) return &d;
    return nullptr;
  }

  // Refill the client's bucket to `now` and return its tokens; a client's
  // first visit starts full (runtime.py:237-248).  Python's min(burst, t)
  // keeps burst unless t < burst; written the same way so a NaN refill
  // (inf budget x 0 s) resolves identically.
  double refill(uint32_t client, double now) {
    if (client >= buckets.size()) buckets.resize(client + 1);
    Bucket& b = buckets[client];
    if (!b.seen) {
      b.seen = true;
      b.tokens = burst;
      b.last = now;
    }
    const double t = b.tokens + budget * (now - b.last);
    b.tokens = (t < burst) ? t : burst;
    b.last = now;
    return b.tokens;
  }

  // Revocations inside the stability window ending at `now` (runtime.py:256-263).
  int64_t churn(Donor& d, double now) {
    const double horizon = now - window;
    while (!d.revocations.empty() && d.revocations.front() < horizon) d.revocations.pop_front();
    return (int64_t)d.revocations.size();
  }

  // select_peer over the donors whose ids are flagged in `take` (indexed like
  // `donors`); -1 when nothing is admissible.
  int select(const std::vector<char>& take, uint64_t size, uint32_t client, double now) {
    bool any = false;
    for (char t : take) any |= (t != 0);
    if (!any) return -1;  // empty candidate list: no bucket refill (runtime.py:171-172)
    if (kind == HV_POLICY_FAIRNESS && !(refill(client, now) >= (double)size)) return -1;
    bool have = false;
    Score best{};
    for (size_t i = 0; i < donors.size(); ++i) {
      if (!take[i]) continue;
      Donor& d = donors[i];
      if (kind == HV_POLICY_STABILITY && !(churn(d, now) < max_revocations)) continue;
      uint64_t used = 0;
      hv_seg_allocated_bytes(d.seg, &used);
      if (used + size > d.ceiling) continue;
      uint64_t leftover = 0, base = 0;
      if (hv_seg_probe(d.seg, size, &leftover, &base) != HV_OK) continue;
      Score s{kind == HV_POLICY_LOCALITY ? d.hops : 0u, leftover, base, d.id};
      if (!have || s < best) {
        best = s;
        have = true;
      }
    }
    return have ? best.dev : -1;
  }
};

HV_EXPORT int hv_placer_create(int policy_kind, double budget_bytes_per_s, double burst_bytes,
                               double stability_window_s, int64_t stability_max_revocations,
                               hv_placer** out) {
  HV_CHECK_ARG(out != nullptr);
  HV_CHECK_ARG(policy_kind >= HV_POLICY_BEST_FIT && policy_kind <= HV_POLICY_STABILITY);
  hv_placer* p = new (std::nothrow) hv_placer();
  if (!p) return HV_E_NOMEM;
  p->kind = policy_kind;
  p->budget = budget_bytes_per_s;
  p->burst = std::isnan(burst_bytes) ? budget_bytes_per_s : burst_bytes;  // burst None -> budget
  p->window = stability_window_s;
  p->max_revocations = stability_max_revocations;
  *out = p;
  return HV_OK;
}

HV_EXPORT int hv_placer_destroy(hv_placer* p) {
  delete p;
  return HV_OK;
}

HV_EXPORT int hv_placer_add_donor(hv_placer* p, int device_id, hv_seg* seg, uint64_t ceiling,
                                  uint32_t hops) {
  HV_CHECK_ARG(p && seg && !p->donor(device_id));
  Donor d;
  d.id = device_id;
  d.seg = seg;
  d.ceiling = ceiling;
  d.hops = hops;
  auto it = p->donors.begin();
  while (it != p->donors.end() && it->id < device_id) ++it;
  p->donors.insert(it, std::move(d));
  return HV_OK;
}

HV_EXPORT int hv_placer_set_ceiling(hv_placer* p, int device_id, uint64_t ceiling) {
  HV_CHECK_ARG(p);
  Donor* d = p->donor(device_id);
  HV_CHECK_ARG(d);
  d->ceiling = ceiling;
  return HV_OK;
}

HV_EXPORT int hv_placer_ceiling(hv_placer* p, int device_id, uint64_t* out) {
  HV_CHECK_ARG(p && out);
  Donor* d = p->donor(device_id);
  HV_CHECK_ARG(d);
  *out = d->ceiling;
  return HV_OK;
}

HV_EXPORT int hv_placer_select(hv_placer* p, uint64_t size, uint32_t client, double now,
                               const int* candidates, int n_candidates, int* device_out) {
  HV_CHECK_ARG(p && device_out && size > 0 && (n_candidates == 0 || candidates));
  std::vector<char> take(p->donors.size(), 0);
  for (int i = 0; i < n_candidates; ++i)
    for (size_t j = 0; j < p->donors.size(); ++j)
      if (p->donors[j].id == candidates[i]) take[j] = 1;
  const int dev = p->select(take, size, client, now);
  *device_out = dev;
  return dev < 0 ? HV_E_NOCAPACITY : HV_OK;
}

HV_EXPORT int hv_placer_alloc(hv_placer* p, uint64_t size, uint32_t client, double now,
                              const int* preferred, int n_preferred, int* device_out,
                              uint64_t* base_out) {
  HV_CHECK_ARG(p && device_out && base_out && size > 0 && (n_preferred == 0 || preferred));
  const size_t n = p->donors.size();
  std::vector<char> pref(n, 0);
  for (int i = 0; i < n_preferred; ++i)
    for (size_t j = 0; j < n; ++j)
      if (p->donors[j].id == preferred[i]) pref[j] = 1;
  int dev;
  if (n_preferred > 0) {
    dev = p->select(pref, size, client, now);
    if (dev < 0) {
      std::vector<char> rest(n);
      for (size_t j = 0; j < n; ++j) rest[j] = !pref[j];
      dev = p->select(rest, size, client, now);
    }
  } else {
    dev = p->select(std::vector<char>(n, 1), size, client, now);
  }
  *device_out = dev;
  if (dev < 0) return HV_E_NOCAPACITY;
  return hv_seg_alloc(p->donor(dev)->seg, size, base_out);
}

HV_EXPORT int hv_placer_spend(hv_placer* p, uint32_t client, uint64_t size, double now) {
  HV_CHECK_ARG(p);
  p->refill(client, now);
  p->buckets[client].tokens -= (double)size;  // runtime.py:252-254
  return HV_OK;
}

HV_EXPORT int hv_placer_tokens(hv_placer* p, uint32_t client, double now, double* out) {
  HV_CHECK_ARG(p && out);
  *out = p->refill(client, now);
  return HV_OK;
}

HV_EXPORT int hv_placer_note_revocation(hv_placer* p, int device_id, double now) {
  HV_CHECK_ARG(p);
  Donor* d = p->donor(device_id);
  HV_CHECK_ARG(d);
  d->revocations.push_back(now);
  return HV_OK;
}

HV_EXPORT int hv_placer_churn(hv_placer* p, int device_id, double now, int64_t* out) {
  HV_CHECK_ARG(p && out);
  Donor* d = p->donor(device_id);
  HV_CHECK_ARG(d);
  *out = p->churn(*d, now);
  return HV_OK;
}
