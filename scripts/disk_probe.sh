#!/bin/bash
# Directory-tier write patterns on the box's disk: new file vs overwrite in place, 1.2 GB, O_DIRECT + fsync.
D=${1:-$GRAFT_REPO_ROOT/gpurun_out/diskprobe}; mkdir -p $D
for i in 1 2 3; do
  echo "new $i: $(dd if=/dev/zero of=$D/new$i bs=16M count=75 oflag=direct conv=fsync 2>&1 | tail -1)"
done
for i in 1 2 3; do
  echo "overwrite $i: $(dd if=/dev/zero of=$D/new$i bs=16M count=75 oflag=direct conv=fsync,notrunc 2>&1 | tail -1)"
done
for i in 1 2 3; do
  echo "trunc-rewrite $i: $(dd if=/dev/zero of=$D/new$i bs=16M count=75 oflag=direct conv=fsync 2>&1 | tail -1)"
done
for i in 1 2 3; do
  echo "read $i: $(dd if=$D/new$i of=/dev/null bs=16M iflag=direct 2>&1 | tail -1)"
done
( time rm -f $D/new1 ) 2>&1 | grep real
rm -rf $D
