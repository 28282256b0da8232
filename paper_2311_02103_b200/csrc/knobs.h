// knobs.h -- experiment knobs, compiled out of the product library.
//
// The product build (python -m paper_2311_02103_b200.build) reads no
// environment variable: every schedule parameter below is its measured
// default.  The experiments build (`--experiments`,
// library under build_exp/, loaded by tools through RELAX_Q4_LIB) defines
// RQ4_EXPERIMENTS: it reads RELAX_Q4_* overrides, records per-CTA timelines
// (RELAX_Q4_TRACE=1, include/relax_q4_debug.h) and links the measured-slower
// decode variants kept under experiments/csrc/.
#pragma once
#include <cstdlib>
#include <cstring>

#ifdef RQ4_EXPERIMENTS
#define RQ4_TRACE 1
namespace rq4 {
inline int knob_int(const char* name, int def) {
    const char* e = std::getenv(name);
    return (e && *e) ? std::atoi(e) : def;
}
inline double knob_double(const char* name, double def) {
    const char* e = std::getenv(name);
    return (e && *e) ? std::atof(e) : def;
}
inline bool knob_is(const char* name, const char* value) {
    const char* e = std::getenv(name);
    return e && std::strcmp(e, value) == 0;
}
}  // namespace rq4
#else
#define RQ4_TRACE 0
namespace rq4 {
inline int knob_int(const char*, int def) { return def; }
inline double knob_double(const char*, double def) { return def; }
inline bool knob_is(const char*, const char*) { return false; }
}  // namespace rq4
#endif
