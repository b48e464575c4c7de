#!/bin/bash
# Build here, then run the given command on the GPU box (only if the build succeeded).
cd /root/repo || exit 1
python -c "import paper_1505_00914_b200._build as b; b.build()" > /tmp/build.log 2>&1 || { tail -20 /tmp/build.log; echo BUILD FAILED; exit 1; }
timeout $((${GPU_TIMEOUT:-1200} + 600)) /usr/local/graft/bin/gpurun --timeout ${GPU_TIMEOUT:-1200} -- "$@"
