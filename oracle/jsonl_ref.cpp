// TEST INFRASTRUCTURE ONLY.  The reference CLI's JSON-lines output, produced the way the CLI
// produces it: nlohmann::json 3.11 (the json.hpp the CLI vendors; a copy ships with the image
// under cudnn_frontend/thirdparty) with record_json / emit_solutions as in
// proj/tools/polypath_main.cpp:125-189, and the reference library's to_decimal / to_double /
// fail_reason_name.  The CLI itself cannot be built here (CLI11 is not vendored), so these two
// functions are restated verbatim in structure around the same library calls.  Built by
// oracle/Makefile as _ref/libjsonref.so; tests/test_jsonl.py compares pp_solutions_jsonl with it.
#include <algorithm>
#include <cstring>
#include <string>
#include <vector>

#include <nlohmann/json.hpp>

#include "pp200.h"
#include "polypath/tracker.hpp"
#include "polypath/xprec_io.hpp"

using json = nlohmann::json;
using namespace polypath;

namespace {

template <class R>
R real_at(const double* p) {
  R v{};
  for (int l = 0; l < precision_traits<R>::limbs; ++l) set_limb(v, l, p[l]);
  return v;
}

int emit(const std::string& o, char* buf, size_t cap, size_t* needed) {
  if (needed) *needed = o.size() + 1;
  if (buf == nullptr || cap < o.size() + 1) return PP_E_CAPACITY;
  std::memcpy(buf, o.c_str(), o.size() + 1);
  return PP_OK;
}

// record_class (polypath_main.cpp:126-131)
const char* record_class(int8_t status, uint8_t reason) {
  if (status == 1) return "converged";
  if (reason == static_cast<uint8_t>(FailReason::diverged)) return "diverged";
  return "failed";
}

template <class R>
std::string solutions(const pp_records* rec, uint32_t dim, const double* gamma, uint64_t seed, const char* command,
                      double wall_ms, uint64_t batches, uint64_t rounds) {
  constexpr int L = precision_traits<R>::limbs;
  std::string out;
  uint64_t converged = 0, diverged = 0, failed = 0;
  std::vector<double> resid;
  for (uint64_t i = 0; i < rec->count; ++i) {
    // record_json (polypath_main.cpp:133-149)
    json jx = json::array();
    for (uint32_t v = 0; v < dim; ++v) {
      const double* z = rec->x + (i * dim + v) * 2 * L;
      jx.push_back({to_decimal(real_at<R>(z)), to_decimal(real_at<R>(z + L))});
    }
    const double res = to_double(real_at<R>(rec->residual + i * L));
    json j;
    j["type"] = "solution";
    j["path"] = rec->path_id[i];
    j["start"] = rec->path_id[i];
    j["x"] = std::move(jx);
    j["residual"] = res;
    j["status"] = record_class(rec->status[i], rec->reason[i]);
    j["annotation"] = fail_reason_name(static_cast<FailReason>(rec->reason[i]));
    j["steps"] = rec->steps[i];
    j["newton"] = rec->newton_iters[i];
    j["rejections"] = rec->rejections[i];
    j["wall_ms"] = wall_ms;
    out += j.dump() + "\n";
    // emit_solutions (polypath_main.cpp:152-189)
    std::string cls = record_class(rec->status[i], rec->reason[i]);
    if (cls == "converged") {
      ++converged;
      resid.push_back(res);
    } else if (cls == "diverged") {
      ++diverged;
    } else {
      ++failed;
    }
  }
  std::sort(resid.begin(), resid.end());
  json s;
  s["type"] = "summary";
  s["command"] = command;
  s["precision"] = precision_traits<R>::name;
  s["gamma"] = {to_double(real_at<R>(gamma)), to_double(real_at<R>(gamma + L))};
  s["seed"] = seed;
  s["paths"] = static_cast<size_t>(rec->count);
  s["converged"] = converged;
  s["diverged"] = diverged;
  s["failed"] = failed;
  if (!resid.empty()) {
    s["residual_min"] = resid.front();
    s["residual_max"] = resid.back();
    s["residual_median"] = resid[resid.size() / 2];
  }
  s["batches"] = batches;
  s["corrector_rounds"] = rounds;
  s["wall_ms"] = wall_ms;
  out += s.dump() + "\n";
  return out;
}

}  // namespace

extern "C" {

int ref_json_doubles(const double* v, size_t n, char* buf, size_t cap, size_t* needed) {
  std::string o;
  for (size_t i = 0; i < n; ++i) o += json(v[i]).dump() + "\n";
  return emit(o, buf, cap, needed);
}

int ref_solutions_jsonl(const pp_records* rec, int prec, uint32_t dim, const double* gamma, uint64_t seed,
                        const char* command, double wall_ms, uint64_t batches, uint64_t rounds, char* buf, size_t cap,
                        size_t* needed) {
  std::string o = prec == PP_D    ? solutions<double>(rec, dim, gamma, seed, command, wall_ms, batches, rounds)
                  : prec == PP_DD ? solutions<DD>(rec, dim, gamma, seed, command, wall_ms, batches, rounds)
                                  : solutions<QD>(rec, dim, gamma, seed, command, wall_ms, batches, rounds);
  return emit(o, buf, cap, needed);
}

}  // extern "C"
