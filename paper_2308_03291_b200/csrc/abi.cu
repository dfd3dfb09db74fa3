// Library-level C-ABI entry points (version, status strings).
#include "common.cuh"

extern "C" int sdb_version(void) { return 100; }  // 0.1.0

extern "C" const char* sdb_status_string(int code) {
  switch (code) {
    case SDB_OK: return "ok";
    case SDB_ERR_ARG: return "invalid argument";
    case SDB_ERR_WORKSPACE: return "workspace missing or too small";
    case SDB_ERR_CUDA: return "CUDA launch error";
    case SDB_ERR_UNSUPPORTED: return "size not supported by this kernel";
    default: return "unknown";
  }
}

// the CUDA runtime's message for the last error an entry point returned
// SDB_ERR_CUDA for ("no error" if none)
extern "C" const char* sdb_last_cuda_error(void) { return cudaGetErrorString((cudaError_t)sdb_last_cuda().load()); }
