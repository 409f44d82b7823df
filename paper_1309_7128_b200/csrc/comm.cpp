// comm.cpp — multi-GPU communicator (strip decomposition); filled in with the NCCL path.
#include "engine.h"

namespace ismgb {
struct Comm {};
void destroy_comm(Comm* c) { delete c; }
}  // namespace ismgb
