// Trace export / replay: the reference's TokenDemand trace file
// ("step,expert,gpu,tokens", proj/src/workload.cpp:175-341,
// proj/include/moesim/workload.hpp:77-86), so device gate histograms
// recorded by this framework can be replayed by the reference engine/CLI and
// reference traces can drive this one.
//
// Same file format and the same acceptance rules as the reference loader:
// header line (a trailing '\r' tolerated), four non-negative integer fields,
// records strictly sorted by (step, expert, gpu), first step 0, equal token
// totals on every step, ids inside explicit dimensions. Errors are
// runtime_error ("<path>:<line>: <what>") -> FM_ERR_RUNTIME, as in the
// reference (workload.cpp:55-58).
#include <algorithm>
#include <cerrno>
#include <cstdlib>
#include <fstream>
#include <sstream>
#include <string>
#include <tuple>
#include <vector>

#include "fm_internal.h"

namespace fm {
namespace {

constexpr const char* kHeader = "step,expert,gpu,tokens";

struct Record {
  long long step, expert, gpu, tokens;
};

[[noreturn]] void fail_at(const std::string& path, int line, const std::string& what) {
  throw std::runtime_error(path + ":" + std::to_string(line) + ": " + what);
}

// One integer field: the whole (non-empty) text must be consumed.
bool parse_field(const std::string& s, long long* v) {
  if (s.empty()) return false;
  errno = 0;
  char* end = nullptr;
  *v = std::strtoll(s.c_str(), &end, 10);
  return errno == 0 && end == s.c_str() + s.size();  // like std::stoll: leading blanks allowed
}

std::vector<Record> read_records(const std::string& path) {
  std::ifstream in(path);
  if (!in) throw std::runtime_error("cannot open trace file: " + path);
  std::string line;
  int no = 1;
  if (!std::getline(in, line)) fail_at(path, 1, "empty trace file");
  if (!line.empty() && line.back() == '\r') line.pop_back();
  if (line != kHeader) fail_at(path, no, "bad header, expected 'step,expert,gpu,tokens'");
  std::vector<Record> recs;
  while (std::getline(in, line)) {
    ++no;
    if (!line.empty() && line.back() == '\r') line.pop_back();
    if (line.empty()) continue;
    long long f[4];
    size_t pos = 0;
    for (int i = 0; i < 4; ++i) {
      const size_t comma = line.find(',', pos);
      if ((i < 3) == (comma == std::string::npos)) fail_at(path, no, "malformed record, expected 4 fields");
      const std::string text = line.substr(pos, comma == std::string::npos ? std::string::npos : comma - pos);
      if (!parse_field(text, &f[i])) fail_at(path, no, "malformed record, bad integer '" + text + "'");
      pos = comma == std::string::npos ? line.size() : comma + 1;
    }
    if (f[3] < 0) fail_at(path, no, "negative token count");
    if (f[0] < 0 || f[1] < 0 || f[2] < 0) fail_at(path, no, "negative id");
    const Record r{f[0], f[1], f[2], f[3]};
    if (!recs.empty()) {
      const Record& p = recs.back();
      if (std::tie(r.step, r.expert, r.gpu) <= std::tie(p.step, p.expert, p.gpu))
        fail_at(path, no, "records not sorted by (step, expert, gpu)");
    }
    recs.push_back(r);
  }
  if (recs.empty()) fail_at(path, no, "trace contains no records");
  return recs;
}

}  // namespace
}  // namespace fm

extern "C" {

int fm_trace_save(const char* path, const int64_t* demand_SNG, const int32_t* step_ids, int num_steps,
                  int num_experts, int num_gpus) {
  return fm::guarded([&] {
    if (!path || (num_steps > 0 && !demand_SNG) || num_steps < 0 || num_experts < 1 || num_gpus < 1)
      throw std::invalid_argument("fm_trace_save: bad arguments");
    std::ostringstream out;
    out << fm::kHeader << '\n';
    const size_t cells = static_cast<size_t>(num_experts) * num_gpus;
    for (int s = 0; s < num_steps; ++s) {
      const int64_t* d = demand_SNG + s * cells;
      const int step = step_ids ? step_ids[s] : s;
      for (int e = 0; e < num_experts; ++e)
        for (int g = 0; g < num_gpus; ++g)
          if (d[static_cast<size_t>(e) * num_gpus + g] != 0)
            out << step << ',' << e << ',' << g << ',' << d[static_cast<size_t>(e) * num_gpus + g] << '\n';
    }
    std::ofstream f(path);
    if (!f) throw std::runtime_error(std::string("cannot open trace file for writing: ") + path);
    f << out.str();
    if (!f) throw std::runtime_error(std::string("failed writing trace file: ") + path);
  });
}

int fm_trace_load(const char* path, int num_experts, int num_gpus, int64_t* demand_SNG,
                  int64_t capacity, int* num_steps_out, int* num_experts_out, int* num_gpus_out) {
  return fm::guarded([&] {
    if (!path) throw std::invalid_argument("fm_trace_load: null path");
    const bool infer = num_experts == 0 && num_gpus == 0;
    if (!infer && (num_experts < 1 || num_gpus < 1))
      throw std::invalid_argument("load_trace: dimensions must be positive");
    const std::string p(path);
    const std::vector<fm::Record> recs = fm::read_records(p);
    long long N = num_experts, G = num_gpus;
    if (infer) {
      N = G = 0;
      for (const fm::Record& r : recs) {
        N = std::max(N, r.expert + 1);
        G = std::max(G, r.gpu + 1);
      }
    }
    if (recs.front().step != 0) throw std::runtime_error(p + ": first step must be 0");
    const long long S = recs.back().step + 1;
    for (const fm::Record& r : recs) {
      if (r.expert >= N) throw std::runtime_error(p + ": expert id " + std::to_string(r.expert) + " out of range");
      if (r.gpu >= G) throw std::runtime_error(p + ": gpu id " + std::to_string(r.gpu) + " out of range");
    }
    std::vector<int64_t> totals(S, 0);
    for (const fm::Record& r : recs) totals[r.step] += r.tokens;
    if (totals[0] <= 0) throw std::runtime_error(p + ": step 0 carries no tokens");
    for (long long s = 0; s < S; ++s)
      if (totals[s] != totals[0])
        throw std::runtime_error(p + ": step " + std::to_string(s) + " total " + std::to_string(totals[s]) +
                                 " does not match step 0 total " + std::to_string(totals[0]));
    if (num_steps_out) *num_steps_out = static_cast<int>(S);
    if (num_experts_out) *num_experts_out = static_cast<int>(N);
    if (num_gpus_out) *num_gpus_out = static_cast<int>(G);
    if (!demand_SNG) return;  // size query
    const int64_t need = S * N * G;
    if (capacity < need)
      throw std::invalid_argument("fm_trace_load: buffer holds " + std::to_string(capacity) + " cells, trace needs " +
                                  std::to_string(need));
    std::fill(demand_SNG, demand_SNG + need, 0);
    for (const fm::Record& r : recs) demand_SNG[(r.step * N + r.expert) * G + r.gpu] = r.tokens;
  });
}

}  // extern "C"
