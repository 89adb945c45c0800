// Exception -> status-code translation for the C ABI.
#pragma once

#include <exception>
#include <string>

#include "../../../include/bfpp.h"
#include "schedule.hpp"

struct bfpp_graph {
    bfpp::TaskGraph g;
};
struct bfpp_timeline {
    bfpp::Timeline tl;
};

namespace bfpp {

ModelSpec to_model(const bfpp_model_spec* m);
ParallelConfig to_config(const bfpp_parallel_config* c);

void set_error(const std::string& msg);

// Runs fn, mapping SpecError -> 2, SimError/any other failure -> 4
// (the reference CLI's exit codes, tools/pipesim.cpp:214-226).
template <class F>
int guarded(F&& fn) {
    try {
        fn();
        return 0;
    } catch (const SpecError& e) {
        set_error(std::string("error[invalid-spec]: ") + e.what());
        return 2;
    } catch (const SimError& e) {
        set_error(std::string("error[simulation]: ") + e.what());
        return 4;
    } catch (const std::exception& e) {
        set_error(std::string("error[execution]: ") + e.what());
        return 4;
    }
}

}  // namespace bfpp
