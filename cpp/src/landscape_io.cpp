// landscape_io.cpp -- report writers and graph export of tunekit/landscape.hpp
// (/root/reference/proj/include/tunekit/landscape.hpp:81-85,96-102;
// SPEC.md:421-426,441-442).  Host-side formatting of results the GPU produced.
#include <algorithm>
#include <charconv>
#include <cmath>
#include <ostream>
#include <string>

#include "tunekit/errors.hpp"
#include "tunekit/landscape.hpp"

namespace tunekit {

namespace {

std::string num(double v) {  // shortest round-trip decimal
    char buf[40];
    const auto r = std::to_chars(buf, buf + sizeof buf, v);
    return std::string(buf, r.ptr);
}

std::string csv_field(const std::string& s) {
    if (s.find_first_of(",\"\n") == std::string::npos) return s;
    std::string q = "\"";
    for (char c : s) {
        if (c == '"') q += '"';
        q += c;
    }
    return q + '"';
}

std::string xml_escape(const std::string& s) {
    std::string o;
    for (char c : s) {
        switch (c) {
            case '&': o += "&amp;"; break;
            case '<': o += "&lt;"; break;
            case '>': o += "&gt;"; break;
            case '"': o += "&quot;"; break;
            default: o += c;
        }
    }
    return o;
}

// Fig. 6 caption: fractions below 0.75 share one flood colour,
// the global minimum is green, [0.75, 1) runs from red to blue.
std::string node_colour(double fraction, bool global_min) {
    if (global_min) return "#00a000";
    if (!(fraction >= 0.75)) return "#c8c8c8";
    const double t = (fraction - 0.75) / 0.25;
    const int r = static_cast<int>(std::lround(220.0 * (1.0 - t)));
    const int b = static_cast<int>(std::lround(220.0 * t));
    char buf[8];
    std::snprintf(buf, sizeof buf, "#%02x30%02x", r, b);
    return buf;
}

}  // namespace

Json centrality_report_to_json(const CentralityReport& report, const SearchSpaceCache& cache) {
    Json j = Json::object();
    Json meta = Json::object();
    meta["kernel"] = cache.metadata().kernel;
    meta["device"] = cache.metadata().device;
    meta["units"] = cache.metadata().units;
    meta["neighbourhood"] = to_string(report.kind);
    meta["damping"] = report.damping;
    meta["dangling_rule"] = "uniform over all nodes";
    meta["minima_rule"] = "ok sinks; fail plateaus excluded";
    meta["p_boundary"] = "p = 0: f <= f_opt; p > 0: f < (1 + p) f_opt";
    j["metadata"] = std::move(meta);
    j["f_opt"] = report.f_opt;
    j["pagerank_iterations"] = report.pagerank_iterations;
    j["pagerank_sum"] = report.pagerank_sum;
    Json mins = Json::array();
    const ParameterSpace& s = cache.space();
    for (const MinimumInfo& m : report.minima) {
        Json e = Json::object();
        e["rank"] = m.rank;
        e["configuration"] = s.key_of(s.config_at(m.rank));
        e["fitness"] = m.fitness;
        e["fraction_of_optimum"] = m.fraction_of_optimum;
        e["pagerank"] = m.pagerank;
        mins.push_back(std::move(e));
    }
    j["minima"] = std::move(mins);
    Json curve = Json::array();
    for (const auto& [p, c] : report.c_p_curve) {
        Json e = Json::object();
        e["p_percent"] = p;
        e["c_p"] = c;
        curve.push_back(std::move(e));
    }
    j["c_p_curve"] = std::move(curve);
    return j;
}

void write_minima_csv(const CentralityReport& report, const SearchSpaceCache& cache,
                      std::ostream& out) {
    const ParameterSpace& s = cache.space();
    out << "rank,configuration,fitness,fraction_of_optimum,pagerank\n";
    for (const MinimumInfo& m : report.minima)
        out << m.rank << ',' << csv_field(s.key_of(s.config_at(m.rank))) << ',' << num(m.fitness)
            << ',' << num(m.fraction_of_optimum) << ',' << num(m.pagerank) << '\n';
}

void write_cp_curve_csv(const CentralityReport& report, std::ostream& out) {
    out << "p_percent,c_p\n";
    for (const auto& [p, c] : report.c_p_curve) out << p << ',' << num(c) << '\n';
}

GraphFormat graph_format_from_string(const std::string& s) {
    std::string t = s;
    std::transform(t.begin(), t.end(), t.begin(), [](unsigned char c) { return std::tolower(c); });
    if (t == "dot") return GraphFormat::Dot;
    if (t == "graphml") return GraphFormat::GraphML;
    if (t == "csv" || t == "edgecsv" || t == "edge-csv") return GraphFormat::EdgeCsv;
    throw InvalidArgument("unknown graph format: " + s + " (expected dot, graphml or csv)");
}

void export_graph(const FitnessFlowGraph& g, const SearchSpaceCache& cache, GraphFormat format,
                  std::ostream& out) {
    const double f_opt = cache.optimum();
    const std::uint32_t n = g.node_count;
    std::vector<std::uint8_t> is_min(n, 0);
    for (std::uint32_t m : g.minima) is_min[m] = 1;
    auto fraction = [&](std::uint32_t u) { return f_opt / g.fitness[u]; };
    auto global = [&](std::uint32_t u) { return is_min[u] && g.fitness[u] == f_opt; };
    if (format == GraphFormat::EdgeCsv) {
        out << "source,target\n";
        for (std::uint32_t u = 0; u < n; ++u)
            for (std::uint64_t i = g.offsets[u]; i < g.offsets[u + 1]; ++i)
                out << u << ',' << g.targets[i] << '\n';
        return;
    }
    if (format == GraphFormat::Dot) {
        out << "digraph ffg {\n  node [shape=circle, style=filled, label=\"\"];\n";
        for (std::uint32_t u = 0; u < n; ++u) {
            out << "  " << u << " [fillcolor=\"" << node_colour(fraction(u), global(u))
                << "\", width=" << (is_min[u] ? "0.5" : "0.2") << ", tooltip=\"f="
                << num(g.fitness[u]) << "\"];\n";
        }
        for (std::uint32_t u = 0; u < n; ++u)
            for (std::uint64_t i = g.offsets[u]; i < g.offsets[u + 1]; ++i)
                out << "  " << u << " -> " << g.targets[i] << ";\n";
        out << "}\n";
        return;
    }
    out << "<?xml version=\"1.0\" encoding=\"UTF-8\"?>\n"
           "<graphml xmlns=\"http://graphml.graphdrawing.org/xmlns\">\n"
           "  <key id=\"fitness\" for=\"node\" attr.name=\"fitness\" attr.type=\"double\"/>\n"
           "  <key id=\"fraction\" for=\"node\" attr.name=\"fraction_of_optimum\" attr.type=\"double\"/>\n"
           "  <key id=\"minimum\" for=\"node\" attr.name=\"local_minimum\" attr.type=\"boolean\"/>\n"
           "  <key id=\"colour\" for=\"node\" attr.name=\"colour\" attr.type=\"string\"/>\n"
           "  <key id=\"size\" for=\"node\" attr.name=\"size\" attr.type=\"double\"/>\n"
           "  <graph id=\"ffg\" edgedefault=\"directed\">\n";
    const ParameterSpace& s = cache.space();
    for (std::uint32_t u = 0; u < n; ++u) {
        out << "    <node id=\"n" << u << "\"><data key=\"fitness\">" << num(g.fitness[u])
            << "</data><data key=\"fraction\">" << num(fraction(u))
            << "</data><data key=\"minimum\">" << (is_min[u] ? "true" : "false")
            << "</data><data key=\"colour\">" << node_colour(fraction(u), global(u))
            << "</data><data key=\"size\">" << (is_min[u] ? "3" : "1") << "</data>"
            << "<!-- " << xml_escape(s.key_of(s.config_at(u))) << " --></node>\n";
    }
    std::uint64_t e = 0;
    for (std::uint32_t u = 0; u < n; ++u)
        for (std::uint64_t i = g.offsets[u]; i < g.offsets[u + 1]; ++i)
            out << "    <edge id=\"e" << e++ << "\" source=\"n" << u << "\" target=\"n"
                << g.targets[i] << "\"/>\n";
    out << "  </graph>\n</graphml>\n";
}

}  // namespace tunekit
