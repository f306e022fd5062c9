#!/bin/bash
# gpurun: concurrent kernel timelines (tools/kernel_trace.py) for several knob settings
# args: "cur" or "env:A=1,B=1"
for v in "$@"; do
  echo "=========== $v"
  ( if [ $v != cur ]; then for kv in $(echo ${v#env:} | tr ',' ' '); do export $kv; done; fi
    timeout 200 python tools/kernel_trace.py 2>&1 | grep -v Warn | grep -v warn | head -45 )
done
