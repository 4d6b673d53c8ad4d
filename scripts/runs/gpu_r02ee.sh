#!/bin/bash
cd ${GRAFT_REPO_ROOT:-.}
O=gpurun_out/r02ee; mkdir -p $O
timeout 2400 python scripts/fullsize_extra.py > $O/fullsize_extra.txt 2>&1; echo "rc=$?" >> $O/fullsize_extra.txt
echo done
