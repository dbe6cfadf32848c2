#!/bin/bash
# run a command under cuda-gdb; if it is still running after $T seconds, interrupt it
# and dump, for CTA 0, each warp's lane-0 PC and registers (gpurun_out/gdb_hang.txt)
T=${T:-25}
cmds=(-ex "set cuda break_on_launch none" -ex "set pagination off" -ex run -ex "info cuda kernels" -ex "info cuda warps")
for w in ${WARPS:-0 4 8 12 13 16 17 18 19 20}; do
  cmds+=(-ex "cuda block 0 warp $w lane 0" -ex "x/2i \$pc" -ex "info registers R2 R3 R5 R6 R8 R9 R22 R23")
done
timeout -s INT $T /usr/local/cuda/bin/cuda-gdb -q -batch "${cmds[@]}" --args "$@" > gpurun_out/gdb_hang.txt 2>&1
echo "gdb rc=$?"; tail -3 gpurun_out/gdb_hang.txt
