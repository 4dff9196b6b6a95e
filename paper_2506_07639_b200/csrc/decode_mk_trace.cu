// Instrumented build of the persistent decode-tick kernel (phase timestamps,
// option "mk_trace"; diagnostic flags, option "mk_flags").  The lean kernel in
// decode_mk.cu dispatches here when either is requested.
#define MK_TRACE 1
#include "decode_mk.cu"
