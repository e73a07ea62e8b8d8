cd "$(dirname "$0")/.."
timeout 600 python tools/determinism.py K:12 30 8
NBBGPU_JIT=0 timeout 600 python tools/determinism.py K:12 30 8
timeout 600 python tools/determinism.py H:11 30 6
timeout 600 python tools/determinism.py C:11 20 6
timeout 600 python tools/determinism.py Y:9 20 6
timeout 600 python tools/determinism.py T:20 20 4
