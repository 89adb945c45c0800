// Timeline exporters and the measured timing model.
//
// * chrome_trace_json — Chrome trace-event JSON of a (simulated or measured) Timeline: one
//   process per device, the three lanes as threads, one complete ("X") event per task in
//   start order, a Transfer mirrored on its receiving device (reference report.cpp:160-212,
//   report.hpp:38-39). Written directly (no JSON library); keys in the reference's (sorted)
//   order and doubles in round-trip precision, so the parsed document equals the reference's.
// * gantt_svg — the reference's SVG Gantt chart (report.cpp:235-290), byte for byte.
// * measured_timing_model — per-kind mean durations of a measured Timeline folded back into
//   the simulator's TimingModel: the simulated replay of the same graph
//   with it shows how much of the measured bubble the schedule itself explains.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <sstream>
#include <tuple>

#include "report.hpp"

namespace bfpp {

namespace {

const char* lane_label(int lane) {
    switch (lane) {
    case 0: return "compute";
    case 1: return "dp-net";
    case 2: return "pp-net";
    }
    return "?";
}

// shortest text that parses back to the same double (JSON number)
std::string json_number(double v) {
    if (!std::isfinite(v)) return "null";
    char buf[40];
    for (int prec = 1; prec <= 17; ++prec) {
        std::snprintf(buf, sizeof buf, "%.*g", prec, v);
        if (std::strtod(buf, nullptr) == v) break;
    }
    std::string s(buf);
    // keep it a JSON float literal when the value is integral ("1000000.0" style)
    if (s.find_first_of(".eEn") == std::string::npos) s += ".0";
    return s;
}

std::string fixed(double v, int decimals) {
    char buf[64];
    std::snprintf(buf, sizeof buf, "%.*f", decimals, v);
    return buf;
}

const char* kind_color(TaskKind k) {
    switch (k) {
    case TaskKind::Fwd: return "#5b9bd5";
    case TaskKind::Bwd: return "#2e5e94";
    case TaskKind::Reduce: return "#e8a33d";
    case TaskKind::Reconstruct: return "#8e5cc7";
    case TaskKind::Transfer: return "#57b894";
    }
    return "#888888";
}

}  // namespace

std::string chrome_trace_json(const Timeline& tl, const TaskGraph& g) {
    std::ostringstream os;
    os << "{\n  \"displayTimeUnit\": \"ms\",\n  \"traceEvents\": [";
    bool first = true;
    auto sep = [&] {
        os << (first ? "\n" : ",\n");
        first = false;
    };
    for (i64 d = 0; d < tl.n_devices; ++d) {
        sep();
        os << "    {\"args\": {\"name\": \"device " << d << "\"}, \"name\": \"process_name\", \"ph\": \"M\", \"pid\": "
           << d << "}";
        for (int lane = 0; lane < 3; ++lane) {
            sep();
            os << "    {\"args\": {\"name\": \"" << lane_label(lane)
               << "\"}, \"name\": \"thread_name\", \"ph\": \"M\", \"pid\": " << d << ", \"tid\": " << lane << "}";
        }
    }
    std::vector<const Task*> order;
    order.reserve(g.tasks.size());
    for (const Task& t : g.tasks) order.push_back(&t);
    std::sort(order.begin(), order.end(), [&](const Task* a, const Task* b) {
        const auto& ea = tl.events[static_cast<size_t>(a->id)];
        const auto& eb = tl.events[static_cast<size_t>(b->id)];
        return std::make_tuple(ea.start, a->device, static_cast<int>(a->lane), a->id) <
               std::make_tuple(eb.start, b->device, static_cast<int>(b->lane), b->id);
    });
    for (const Task* t : order) {
        const auto& ev = tl.events[static_cast<size_t>(t->id)];
        const std::string body = std::string("\"dur\": ") + json_number((ev.end - ev.start) * 1e6) + ", \"name\": \"" +
                                 kind_name(t->kind) + " mb" + std::to_string(t->micro_batch) + " s" +
                                 std::to_string(t->stage) + "\", \"ph\": \"X\", \"pid\": ";
        const std::string tail = ", \"tid\": " + std::to_string(static_cast<int>(t->lane)) +
                                 ", \"ts\": " + json_number(ev.start * 1e6) + "}";
        sep();
        os << "    {" << body << t->device << tail;
        if (t->kind == TaskKind::Transfer) {  // mirrored on the receiving device
            sep();
            os << "    {" << body << t->peer_device << tail;
        }
    }
    os << (first ? "]\n}\n" : "\n  ]\n}\n");
    return os.str();
}

std::string gantt_svg(const Timeline& tl, const TaskGraph& g) {
    const double width = 1000.0, row_h = 14.0, left = 70.0, top = 10.0;
    const double span = std::max(tl.makespan, 1e-12);
    const double scale = (width - left - 10.0) / span;
    const i64 rows = tl.n_devices * 3;
    const double height = top * 2 + row_h * static_cast<double>(rows);
    std::ostringstream os;
    os << "<svg xmlns=\"http://www.w3.org/2000/svg\" width=\"" << width << "\" height=\"" << height << "\">\n";
    os << "<rect width=\"100%\" height=\"100%\" fill=\"white\"/>\n";
    for (i64 d = 0; d < tl.n_devices; ++d)
        for (int l = 0; l < 3; ++l) {
            const double y = top + row_h * static_cast<double>(d * 3 + l);
            os << "<text x=\"2\" y=\"" << fixed(y + row_h - 4, 1) << "\" font-size=\"9\" font-family=\"monospace\">d"
               << d << " " << lane_label(l) << "</text>\n";
        }
    std::vector<const Task*> order;
    for (const Task& t : g.tasks) order.push_back(&t);
    std::sort(order.begin(), order.end(), [](const Task* a, const Task* b) { return a->id < b->id; });
    for (const Task* t : order) {
        const auto& ev = tl.events[static_cast<size_t>(t->id)];
        const double w = std::max((ev.end - ev.start) * scale, 0.5);
        auto draw = [&](i64 device) {
            const double x = left + ev.start * scale;
            const double y = top + row_h * static_cast<double>(device * 3 + static_cast<int>(t->lane));
            os << "<rect x=\"" << fixed(x, 2) << "\" y=\"" << fixed(y + 1, 2) << "\" width=\"" << fixed(w, 2)
               << "\" height=\"" << fixed(row_h - 2, 2) << "\" fill=\"" << kind_color(t->kind)
               << "\" stroke=\"#333333\" stroke-width=\"0.2\"><title>" << kind_name(t->kind) << " mb"
               << t->micro_batch << " s" << t->stage << "</title></rect>\n";
        };
        draw(t->device);
        if (t->kind == TaskKind::Transfer) draw(t->peer_device);
    }
    os << "</svg>\n";
    return os.str();
}

TimingModel measured_timing_model(const TaskGraph& g, const Timeline& tl) {
    double sum[5] = {}, cnt[5] = {};
    for (const Task& t : g.tasks) {
        const auto& ev = tl.events[static_cast<size_t>(t.id)];
        const double d = ev.end - ev.start;
        if (!std::isfinite(d)) continue;
        const int k = static_cast<int>(t.kind);
        sum[k] += d;
        cnt[k] += 1;
    }
    auto mean = [&](TaskKind k) {
        const int i = static_cast<int>(k);
        return cnt[i] > 0 ? sum[i] / cnt[i] : 0.0;
    };
    TimingModel tm;
    tm.t_fwd_stage = mean(TaskKind::Fwd);
    if (tm.t_fwd_stage <= 0) throw SimError("measured_timing_model: the timeline has no forward task durations");
    tm.bwd_ratio = cnt[static_cast<int>(TaskKind::Bwd)] > 0 ? mean(TaskKind::Bwd) / tm.t_fwd_stage : 2.0;
    tm.t_pp_transfer = mean(TaskKind::Transfer);
    tm.pp_latency = 0.0;  // folded into the measured transfer durations
    tm.t_dp_reduce_stage = mean(TaskKind::Reduce);
    tm.t_dp_reconstruct_stage = mean(TaskKind::Reconstruct);
    return tm;
}

}  // namespace bfpp
