// pswa/threading.h — the reference's host worker API (drop-in for
// proj/include/pswa/threading.h:24-31, same names and contract). Backed by a
// persistent pool (csrc/host/threading.cpp) instead of threads spawned per
// call. Index-partitioned: fn(i) runs exactly once per index, so results do
// not depend on the worker count. The device path does not use it; it serves
// reference-side host code (container I/O, oracle-style loops) next to it.
#ifndef PSWA_THREADING_H_
#define PSWA_THREADING_H_

#include <cstdint>
#include <functional>

namespace pswa {

// Defaults to PSWA_THREADS when set, else 1.
void set_workers(int n);
int workers();
void parallel_for(int64_t begin, int64_t end, const std::function<void(int64_t)>& fn);

}  // namespace pswa

#endif  // PSWA_THREADING_H_
