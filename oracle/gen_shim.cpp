// gen_shim.cpp -- TEST INFRASTRUCTURE ONLY.  Error plumbing for the standalone build of the
// shared input generator (paper_2203_08498_b200/csrc/generators.cpp compiled by g++ into
// oracle/libgen_host.so), so the oracle harness and bench.py's reference arm generate the
// BASELINE.json inputs without mapping librcg_b200.so.  Same arrays, bit for bit: one source.
#include <string>

namespace rcg {
static thread_local std::string g_gen_error;
void set_error(const std::string& msg) { g_gen_error = msg; }
void clear_error() { g_gen_error.clear(); }
}  // namespace rcg

extern "C" const char* gen_last_error(void) { return rcg::g_gen_error.c_str(); }
