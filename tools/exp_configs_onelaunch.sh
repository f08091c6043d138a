# Multi-pass BASELINE configs through the one-launch frame path (what render() runs).
export SRT_ONE_LAUNCH=1
echo "C2 100k 512x512 16spp N=1: $(timeout 300 python tools/time_frames.py 100000 512 512 16 1 10 2>&1 | tail -1 | cut -c1-120)"
echo "1M 1080p 16spp N=1: $(timeout 300 python tools/time_frames.py 1000000 1920 1080 16 1 5 2>&1 | tail -1 | cut -c1-120)"
echo "C4 3M 3840x2160 4spp N=1: $(timeout 300 python tools/time_frames.py 3000000 3840 2160 4 1 5 2>&1 | tail -1 | cut -c1-120)"
echo "C5 6M 1080p 1024spp N=1: $(timeout 600 python tools/time_frames.py 6000000 1920 1080 1024 1 2 2>&1 | tail -1 | cut -c1-120)"
