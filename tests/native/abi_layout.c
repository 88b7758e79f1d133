/* Prints sizeof/offsetof of every tvgpu.h struct: tests/test_native_abi.py compares them
 * with the numpy structured dtypes the ctypes binding uses. */
#include <stddef.h>
#include <stdio.h>
#include "tvgpu.h"

#define F(T, f) printf("%s.%s %zu\n", #T, #f, offsetof(T, f))
int main(void) {
  printf("tv_array_box %zu\n", sizeof(tv_array_box));
  F(tv_array_box, base); F(tv_array_box, shape); F(tv_array_box, off);
  printf("tv_copy %zu\n", sizeof(tv_copy));
  F(tv_copy, src); F(tv_copy, dst); F(tv_copy, ext); F(tv_copy, rank); F(tv_copy, itemsize);
  F(tv_copy, src_dtype); F(tv_copy, dst_dtype); F(tv_copy, flags);
  printf("tv_write_item %zu\n", sizeof(tv_write_item));
  F(tv_write_item, src); F(tv_write_item, ext); F(tv_write_item, rank); F(tv_write_item, itemsize);
  F(tv_write_item, file); F(tv_write_item, device); F(tv_write_item, file_off);
  printf("tv_output %zu\n", sizeof(tv_output));
  F(tv_output, path); F(tv_output, host); F(tv_output, size);
  printf("tv_read_item %zu\n", sizeof(tv_read_item));
  F(tv_read_item, input); F(tv_read_item, device); F(tv_read_item, in_off); F(tv_read_item, nbytes);
  F(tv_read_item, direct_dst); F(tv_read_item, first_copy); F(tv_read_item, n_copies);
  printf("tv_input %zu\n", sizeof(tv_input));
  printf("tv_stats %zu\n", sizeof(tv_stats));
  F(tv_stats, bytes_device); F(tv_stats, seconds_total); F(tv_stats, seconds_kernel);
  F(tv_stats, seconds_io); F(tv_stats, seconds_wait_dma); F(tv_stats, seconds_wait_slot);
  F(tv_stats, recycled_files); F(tv_stats, zero_copy_bytes); F(tv_stats, registered_files);
  return 0;
}
