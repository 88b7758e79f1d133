set -x
timeout 600 tools/tma2d_pack_probe > gpurun_out/r2_tma2d_pack.jsonl 2> gpurun_out/r2_tma2d_pack.err; echo probe rc=$?
