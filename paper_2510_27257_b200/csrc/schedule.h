// Schedule generator internals (see schedule.cpp).
#pragma once

#include <array>
#include <memory>
#include <string>
#include <vector>

#include "stp.h"

namespace stp {

struct Schedule {
  int kind = 0, pp = 1, vpp = 2, tp = 1, m = 1;
  std::vector<std::vector<stp_action>> ranks;  // per PP rank
};

int sched_n_vstages(int kind, int p);
int sched_n_chunks(int kind);
int sched_vstage(int kind, int p, int d, int c);
int sched_vstage_device(int kind, int p, int vs);
stp_status schedule_build(int p, int vpp, int tp, int m, int kind, Schedule& s);
stp_status schedule_expand(const Schedule& s, int d, const std::vector<int>& lay, std::vector<stp_unit>& units,
                           bool vit_first = false);
int schedule_stash_slots(const Schedule& s, int d);
std::string schedule_text(const Schedule& s, const int* lay, bool vit_first = false);
stp_status layer_split(int n_layers, int n_slots, int* out);

}  // namespace stp
