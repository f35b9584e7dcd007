#!/bin/sh
# usage: tools/g.sh <name> '<command>'   (runs on the GPU box from the repo root)
cd /root/repo || exit 1
name=$1; shift
timeout 2400 /usr/local/graft/bin/gpurun --timeout 1500 -- "$@" > gpurun_out/call_$name.log 2>&1
tail -2 gpurun_out/call_$name.log
