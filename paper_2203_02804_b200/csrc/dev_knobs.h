// Development A/B knobs.
//
// The shipped library (`make`, libttpricer_b200.so) reads no environment
// variable: every knob below compiles to its default, so the GPU suite, the
// smoke test and the benchmark all run exactly one code path per block shape.
// `make dev` builds libttpricer_b200_dev.so with -DTTP_DEV, where each knob
// reads its TTP_* variable once per process; only the A/B tools and the
// knob-neutrality tests (tests/test_dev_knobs_gpu.py) load that library.
#pragma once

#include <cstdlib>

#ifdef TTP_DEV
inline const char* ttp_dev_env(const char* name) { return std::getenv(name); }
#else
inline const char* ttp_dev_env(const char*) { return nullptr; }
#endif
