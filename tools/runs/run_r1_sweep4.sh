#!/bin/bash
# Engine sizing sweep under torchrun on all visible GPUs (C2, 8 layers): save/restore GB/s
# against the storage probe, one JSON summary line per setting.
cd "$(dirname "$0")/../.."
N=$(python -c "import torch;print(torch.cuda.device_count())")
{ nproc; free -g; lscpu | grep -i "cache\|numa"; } > gpurun_out/sw${N}_probe.log 2>&1
run() {
  tag=$1; shift
  env "$@" timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 \
    --master-port 29611 bench.py --gpus $N --layers ${LAYERS:-8} --steps 2 --warmup 2 --no-e2e --no-cpu-baseline \
    > gpurun_out/sw${N}_$tag.log 2>&1
  python - "$tag" "gpurun_out/sw${N}_$tag.log" "$*" <<'PY' >> gpurun_out/sw${N}.jsonl
import json, sys
tag, path, env = sys.argv[1:4]
line = [l for l in open(path) if l.startswith("{")]
if not line:
    print(json.dumps({"tag": tag, "env": env, "error": open(path).read()[-300:]})); sys.exit()
d = json.loads(line[-1]); r = d["io_roofline"]
print(json.dumps({"tag": tag, "env": env, "value": d["value"], "save": d["save_GBps"], "restore": d["restore_GBps"],
  "w_probe": r["storage_write_GBps"], "r_probe": r["storage_read_GBps"], "eng": d["engine_rank0"]}))
PY
  tail -1 gpurun_out/sw${N}.jsonl | cut -c1-200
}
run default
run slot512k TVGPU_SLOT_BYTES=524288
run slot512k_s32 TVGPU_SLOT_BYTES=524288 TVGPU_SLOTS=32
run thr4 TVGPU_THREADS=4
run thr10 TVGPU_THREADS=10
run slot4m TVGPU_SLOT_BYTES=4194304 TVGPU_SLOTS=8
run default2
