// oracle/ref_synth_glue.cpp — TEST INFRASTRUCTURE: input generation for the
// reference arm.
//
// oracle/Makefile compiles the product's HOST generator source
// (paper_1002_1168_b200/csrc/synth.cpp, integer-only, no CUDA) into
// oracle/_ref/libme_ref.so with its two entry points renamed to
// ref_synth_preset / ref_synth, so bench.py's reference arm builds the very
// same input bytes without loading libme_b200.so.  It produces inputs only;
// nothing generated here is timed or compared.
#include <string>

#include "me_b200.h"

namespace {
thread_local std::string g_synth_err;
}

// The generator reports errors through me_fail (me_internal.h).
me_status me_fail(me_status code, const std::string& msg) {
    g_synth_err = msg;
    return code;
}

extern "C" const char* ref_synth_last_error(void) { return g_synth_err.c_str(); }
