// Timing tables, CSV I/O and the Eq. 5 batch step: SPEC.md:326-398.
#include "streamtune/dataset.hpp"

#include <algorithm>
#include <cerrno>
#include <cmath>
#include <cstdlib>
#include <iomanip>
#include <limits>
#include <map>
#include <sstream>

namespace streamtune {
namespace {

std::string trim(const std::string& s) {
  std::size_t b = 0, e = s.size();
  while (b < e && (s[b] == ' ' || s[b] == '\t' || s[b] == '\r' || s[b] == '\n')) ++b;
  while (e > b && (s[e - 1] == ' ' || s[e - 1] == '\t' || s[e - 1] == '\r' || s[e - 1] == '\n')) --e;
  return s.substr(b, e - b);
}

std::vector<std::string> split_commas(const std::string& line) {
  std::vector<std::string> out;
  std::string cell;
  std::istringstream ss(line);
  while (std::getline(ss, cell, ',')) out.push_back(trim(cell));
  if (!line.empty() && line.back() == ',') out.push_back("");
  return out;
}

double parse_real(const std::string& s, std::size_t line, const std::string& col) {
  if (s.empty()) throw MalformedRowError(line, col, "empty value");
  errno = 0;
  char* end = nullptr;
  const double v = std::strtod(s.c_str(), &end);
  if (end != s.c_str() + s.size() || errno == ERANGE)
    throw MalformedRowError(line, col, "not a number: '" + s + "'");
  if (!std::isfinite(v)) throw MalformedRowError(line, col, "non-finite value");
  return v;
}

std::uint64_t parse_size(const std::string& s, std::size_t line, const std::string& col) {
  const double v = parse_real(s, line, col);
  if (v < 1.0 || v != std::floor(v) || v > 9.0e18)
    throw MalformedRowError(line, col, "SLAE size must be a positive integer: '" + s + "'");
  return static_cast<std::uint64_t>(v);
}

// Reads non-blank lines; checks the header; returns (line number, cells).
std::vector<std::pair<std::size_t, std::vector<std::string>>> read_csv(
    std::istream& in, const std::vector<std::string>& header) {
  std::vector<std::pair<std::size_t, std::vector<std::string>>> rows;
  std::string line;
  std::size_t lineno = 0;
  bool seen_header = false;
  while (std::getline(in, line)) {
    ++lineno;
    const std::string t = trim(line);
    if (t.empty()) continue;
    auto cells = split_commas(t);
    if (!seen_header) {
      if (cells != header) {
        std::string want;
        for (const auto& h : header) want += (want.empty() ? "" : ",") + h;
        throw MalformedRowError(lineno, "header", "expected header '" + want + "'");
      }
      seen_header = true;
      continue;
    }
    if (cells.size() != header.size())
      throw MalformedRowError(lineno, cells.size() < header.size() ? header[cells.size()] : "extra",
                              "expected " + std::to_string(header.size()) + " columns");
    rows.emplace_back(lineno, std::move(cells));
  }
  if (!seen_header) throw MalformedRowError(lineno, "header", "missing header");
  return rows;
}

const std::vector<std::string> kStageHeader = {"slae_size", "t1_h2d", "t1_comp", "t1_d2h",
                                               "t2_comp",   "t3_h2d", "t3_comp", "t3_d2h"};
const std::vector<std::string> kRunHeader = {"slae_size", "num_streams", "t_str"};

std::string full(double v) {
  std::ostringstream s;
  s << std::setprecision(17) << v;
  return s.str();
}

}  // namespace

const StageTimings* StageTimingsTable::find(std::uint64_t slae_size) const {
  auto it = std::lower_bound(rows.begin(), rows.end(), slae_size,
                             [](const StageTimings& r, std::uint64_t s) { return r.slae_size < s; });
  if (it != rows.end() && it->slae_size == slae_size) return &*it;
  return nullptr;
}

StageTimingsTable load_stage_timings(std::istream& in) {
  StageTimingsTable t;
  std::map<std::uint64_t, StageTimings> seen;
  for (auto& [line, cells] : read_csv(in, kStageHeader)) {
    StageTimings st;
    st.slae_size = parse_size(cells[0], line, kStageHeader[0]);
    double* fields[7] = {&st.t1_h2d, &st.t1_comp, &st.t1_d2h, &st.t2_comp,
                         &st.t3_h2d, &st.t3_comp, &st.t3_d2h};
    for (int k = 0; k < 7; ++k) {
      *fields[k] = parse_real(cells[k + 1], line, kStageHeader[k + 1]);
      if (*fields[k] < 0.0) throw NegativeDurationError(line, kStageHeader[k + 1]);
    }
    if (seen.count(st.slae_size)) throw DuplicateSizeError(st.slae_size);
    seen.emplace(st.slae_size, st);
  }
  for (auto& kv : seen) t.rows.push_back(kv.second);
  return t;
}

StreamedRunTable load_streamed_runs(std::istream& in) {
  StreamedRunTable t;
  std::map<std::pair<std::uint64_t, int>, bool> seen;
  for (auto& [line, cells] : read_csv(in, kRunHeader)) {
    const std::uint64_t size = parse_size(cells[0], line, kRunHeader[0]);
    const double nd = parse_real(cells[1], line, kRunHeader[1]);
    if (nd != std::floor(nd) || std::fabs(nd) > 1e9)
      throw MalformedRowError(line, kRunHeader[1], "stream count must be an integer");
    const int n = static_cast<int>(nd);
    StreamCount sc(n);  // throws InvalidStreamCountError
    const double t_str = parse_real(cells[2], line, kRunHeader[2]);
    if (t_str < 0.0) throw NegativeDurationError(line, kRunHeader[2]);
    if (seen.count({size, n})) throw DuplicateSizeError(size, n);
    seen[{size, n}] = true;
    t.rows.push_back(StreamedRun{size, sc, t_str});
  }
  return t;
}

void save_stage_timings(std::ostream& out, const StageTimingsTable& t) {
  for (std::size_t k = 0; k < kStageHeader.size(); ++k) out << (k ? "," : "") << kStageHeader[k];
  out << "\n";
  for (const StageTimings& r : t.rows)
    out << r.slae_size << "," << full(r.t1_h2d) << "," << full(r.t1_comp) << "," << full(r.t1_d2h)
        << "," << full(r.t2_comp) << "," << full(r.t3_h2d) << "," << full(r.t3_comp) << ","
        << full(r.t3_d2h) << "\n";
}

void save_streamed_runs(std::ostream& out, const StreamedRunTable& t) {
  out << "slae_size,num_streams,t_str\n";
  for (const StreamedRun& r : t.rows)
    out << r.slae_size << "," << r.num_streams.value() << "," << full(r.t_str) << "\n";
}

std::vector<OverheadRow> derive_overhead_rows(const StageTimingsTable& stage,
                                              const StreamedRunTable& runs) {
  std::vector<OverheadRow> out;
  for (const StreamedRun& r : runs.rows) {
    const StageTimings* st = stage.find(r.slae_size);
    if (!st) throw MissingStageTimingsError(r.slae_size);
    if (r.num_streams.value() < 2) continue;  // n = 1 calibrates T_non_str only
    const double ovh =
        overhead_from_measurement(r.t_str, total_unstreamed(*st), r.num_streams, overlap_sum(*st));
    out.push_back(OverheadRow{r.slae_size, r.num_streams.value(), ovh});
  }
  return out;
}

// ---- transcriptions of PAPER.md tables -----------------------------------

const std::vector<ReferenceData::Table1Row>& ReferenceData::table1() {
  static const std::vector<Table1Row> t = {
      {4000, 0.221312, 0.014848, 0.006592, 0.030688, 0.273440, 7.8, 1},
      {40000, 0.216544, 0.057312, 0.015456, 0.038112, 0.327424, 8.6, 1},
      {400000, 0.393184, 0.402944, 0.102784, 0.205408, 1.104320, 15.8, 4},
      {4000000, 1.993980, 3.897410, 0.975392, 2.130500, 8.997282, 45.0, 32},
      {40000000, 17.451500, 38.836800, 9.606720, 20.981600, 86.876620, 139.8, 32},
  };
  return t;
}

const std::vector<ReferenceData::Table2Row>& ReferenceData::table2() {
  static const std::vector<Table2Row> t = {
      {2, 7.999136, 8.817440, 2.433568, 0.398480, 0.818304},
      {4, 7.533248, 8.817440, 2.433568, 0.540984, 1.284192},
      {8, 7.401472, 8.817440, 2.433568, 0.713404, 1.415968},
      {16, 7.445952, 8.817440, 2.433568, 0.909982, 1.371488},
      {32, 7.599968, 8.817440, 2.433568, 1.140047, 1.217472},
  };
  return t;
}

const std::vector<ReferenceData::Table4Row>& ReferenceData::table4() {
  static const std::vector<Table4Row> t = {
      {1000, 1, 1},        {4000, 1, 1},        {5000, 1, 1},        {8000, 1, 1},
      {10000, 1, 1},       {40000, 1, 1},       {50000, 1, 1},       {80000, 1, 1},
      {100000, 1, 2},      {400000, 4, 4},      {500000, 8, 4},      {800000, 8, 8},
      {1000000, 8, 8},     {2500000, 16, 16},   {4000000, 32, 32},   {5000000, 32, 32},
      {7500000, 32, 32},   {8000000, 32, 32},   {10000000, 32, 32},  {25000000, 32, 32},
      {40000000, 32, 32},  {50000000, 32, 32},  {75000000, 32, 32},  {80000000, 32, 32},
      {100000000, 32, 32},
  };
  return t;
}

const std::vector<ReferenceData::Table5Row>& ReferenceData::table5() {
  static const std::vector<Table5Row> t = {
      {0, 1, 1, false},          {400000, 2, 4, true},      {500000, 4, 8, true},
      {800000, 8, 8, false},     {1000000, 4, 8, true},     {2500000, 16, 16, false},
      {4000000, 16, 32, true},   {5000000, 16, 32, true},   {7500000, 32, 32, false},
      {8000000, 32, 32, false},  {10000000, 16, 32, true},  {25000000, 16, 32, true},
      {40000000, 32, 32, false}, {50000000, 32, 32, false}, {75000000, 32, 32, false},
      {80000000, 32, 32, false}, {100000000, 32, 32, false},
  };
  return t;
}

}  // namespace streamtune
