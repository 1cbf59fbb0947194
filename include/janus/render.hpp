// janus/render.hpp — timeline rendering (simulator `render`)
// of measured (executor CUDA-event timeline) or replayed (graph.hpp:168)
// schedules: ASCII (one row per device, one column per time quantum, the
// phase name at the start of each instruction, '=' while it runs, '.' for a
// bubble) and a self-contained SVG (device lanes, rectangles coloured by
// phase, time axis).  Byte-for-byte deterministic for a given input.
#pragma once

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <string>
#include <vector>

#include "janus/errors.hpp"
#include "janus/graph.hpp"
#include "janus/ir.hpp"

namespace janus {
namespace render {

/// One compute span: phase 0 FE, 1 FF, 2 BE, 3 BF (the ir.hpp:17 phase index).
struct Span {
  int device = 0, phase = 0, micro_batch = 0;
  double start = 0, end = 0;
};

inline const char* phase_name(int p) {
  static const char* n[4] = {"FE", "FF", "BE", "BF"};
  return (p >= 0 && p < 4) ? n[p] : "??";
}

/// Compute spans of a replayed schedule.
inline std::vector<Span> spans_of(const DepGraph& g, const ReplayResult& r) {
  std::vector<Span> out;
  for (int i = 0; i < g.size(); ++i) {
    const Instruction& in = *g.flat[static_cast<std::size_t>(i)];
    int p = -1;
    switch (in.kind) {
      case InstrKind::FE: p = 0; break;
      case InstrKind::FF: p = 1; break;
      case InstrKind::BE: p = 2; break;
      case InstrKind::BF: p = 3; break;
      default: break;
    }
    if (p < 0) continue;
    out.push_back(Span{in.device, p, in.micro_batch, r.start[static_cast<std::size_t>(i)], r.end[static_cast<std::size_t>(i)]});
  }
  return out;
}

/// quantum <= 0: automatic, half the shortest span (every name fits).
inline std::string ascii(std::vector<Span> spans, double quantum) {
  if (spans.empty()) return "";
  if (!(quantum > 0)) {
    double m = 0;
    for (const Span& s : spans)
      if (s.end > s.start && (m == 0 || s.end - s.start < m)) m = s.end - s.start;
    quantum = m > 0 ? m / 2 : 1.0;
  }
  double t0 = spans[0].start, t1 = spans[0].end;
  int D = 0;
  for (const Span& s : spans) {
    t0 = std::min(t0, s.start);
    t1 = std::max(t1, s.end);
    D = std::max(D, s.device + 1);
  }
  const int W = std::max(1, static_cast<int>(std::ceil((t1 - t0) / quantum - 1e-9)));
  if (W > 100000) throw domain_error("render: more than 100000 columns; raise the quantum");
  std::vector<std::string> rows(static_cast<std::size_t>(D), std::string(static_cast<std::size_t>(W), '.'));
  std::stable_sort(spans.begin(), spans.end(), [](const Span& a, const Span& b) { return a.start < b.start; });
  for (const Span& s : spans) {
    std::string& row = rows[static_cast<std::size_t>(s.device)];
    const int a = std::clamp(static_cast<int>(std::floor((s.start - t0) / quantum + 1e-9)), 0, W - 1);
    const int b = std::clamp(static_cast<int>(std::ceil((s.end - t0) / quantum - 1e-9)), a + 1, W);
    const char* nm = phase_name(s.phase);
    for (int c = a; c < b; ++c) row[static_cast<std::size_t>(c)] = c - a < 2 ? nm[c - a] : '=';
  }
  std::string out;
  for (int d = 0; d < D; ++d) out += "D" + std::to_string(d) + " |" + rows[static_cast<std::size_t>(d)] + "|\n";
  return out;
}

inline std::string svg(const std::vector<Span>& spans, double px_per_unit = 1.0) {
  static const char* colour[4] = {"#4e79a7", "#59a14f", "#f28e2b", "#e15759"};
  double t0 = 0, t1 = 0;
  int D = 0;
  bool first = true;
  for (const Span& s : spans) {
    t0 = first ? s.start : std::min(t0, s.start);
    t1 = first ? s.end : std::max(t1, s.end);
    first = false;
    D = std::max(D, s.device + 1);
  }
  const double lane = 24, left = 40, W = left + (t1 - t0) * px_per_unit + 10, Hh = lane * D + 30;
  char buf[256];
  std::string out;
  std::snprintf(buf, sizeof buf,
                "<svg xmlns=\"http://www.w3.org/2000/svg\" width=\"%.1f\" height=\"%.1f\" font-family=\"monospace\" font-size=\"10\">\n",
                W, Hh);
  out += buf;
  for (int d = 0; d < D; ++d) {
    std::snprintf(buf, sizeof buf, "<text x=\"2\" y=\"%.1f\">D%d</text>\n", lane * d + 16, d);
    out += buf;
  }
  for (const Span& s : spans) {
    std::snprintf(buf, sizeof buf,
                  "<rect x=\"%.2f\" y=\"%.1f\" width=\"%.2f\" height=\"%.1f\" fill=\"%s\"><title>%s mb=%d</title></rect>\n",
                  left + (s.start - t0) * px_per_unit, lane * s.device + 4, std::max(0.5, (s.end - s.start) * px_per_unit),
                  lane - 8, colour[std::clamp(s.phase, 0, 3)], phase_name(s.phase), s.micro_batch);
    out += buf;
  }
  std::snprintf(buf, sizeof buf, "<line x1=\"%.1f\" y1=\"%.1f\" x2=\"%.1f\" y2=\"%.1f\" stroke=\"black\"/>\n", left,
                lane * D + 6, W - 10, lane * D + 6);
  out += buf;
  std::snprintf(buf, sizeof buf, "<text x=\"%.1f\" y=\"%.1f\">0</text><text x=\"%.1f\" y=\"%.1f\">%.6g</text>\n", left,
                lane * D + 20, W - 60, lane * D + 20, t1 - t0);
  out += buf;
  out += "</svg>\n";
  return out;
}

}  // namespace render
}  // namespace janus
