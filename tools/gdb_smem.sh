#!/bin/bash
# run a command under cuda-gdb; after $T s interrupt and dump CTA ${BLK:-0}'s shared words at $ADDR
T=${T:-40}
cmds=(-ex "set cuda break_on_launch none" -ex "set pagination off" -ex run -ex "info cuda kernels"
      -ex "cuda block ${BLK:-0} warp 0 lane 0" -ex "x/${N:-160}xw (@shared unsigned int*)${ADDR:-0x34400}")
timeout -s INT $T /usr/local/cuda/bin/cuda-gdb -q -batch "${cmds[@]}" --args "$@" > gpurun_out/gdb_smem.txt 2>&1
echo "gdb rc=$?"; grep -A60 'shared' gpurun_out/gdb_smem.txt | head -70
