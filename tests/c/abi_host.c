/* Plain-C consumer of the C-ABI (include/fastcdf_b200.h): links libfastcdf_b200.so, checks the
 * ABI version, queries a workspace size (host arithmetic only, no device touched) and reads the
 * thread-local error message of a rejected call.  Built and run by tests/test_abi_host.py. */
#include <stdio.h>
#include <string.h>

#include "fastcdf_b200.h"

int main(void) {
  if (fcg_abi_version() != FCG_ABI_VERSION) {
    fprintf(stderr, "abi version mismatch\n");
    return 1;
  }
  int64_t m[3] = {512, 512, 512};
  int32_t delta[3] = {1, -1, 1};
  size_t bytes = 0;
  int rc = fcg_ecdf_grid(NULL, 1000, 3, NULL, NULL, m, delta, 0, 1, 0, NULL, NULL, &bytes, NULL);
  if (rc != FCG_OK || bytes < (size_t)512 * 512 * 512 * 4) {
    fprintf(stderr, "workspace query failed: rc=%d bytes=%zu\n", rc, bytes);
    return 2;
  }
  int64_t m9[9] = {2, 2, 2, 2, 2, 2, 2, 2, 2};
  int32_t d9[9] = {1, 1, 1, 1, 1, 1, 1, 1, 1};
  rc = fcg_ecdf_grid(NULL, 10, 9, NULL, NULL, m9, d9, 0, 1, 0, NULL, NULL, &bytes, NULL);
  if (rc == FCG_OK || strstr(fcg_last_error(), "dimension") == NULL) {
    fprintf(stderr, "expected a dimension error, got rc=%d '%s'\n", rc, fcg_last_error());
    return 3;
  }
  printf("abi %d ok, workspace %zu bytes\n", fcg_abi_version(), bytes);
  return 0;
}
