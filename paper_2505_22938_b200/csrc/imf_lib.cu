// imf_lib.cu -- single translation unit for the extension (kernels and their
// host launch stubs must live in the same TU without -rdc).
#include "imf_sort.cu"
#include "imf_grank.cu"
#include "imf_select.cu"
#include "imf_pair.cu"
#include "imf_direct.cu"
#include "imf_api.cu"
#include "imf_peak.cu"
