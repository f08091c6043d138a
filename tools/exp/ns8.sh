for c in 0 7 8; do echo -n "N=8 cfg $c "; SRT_PACKET_CFG=$c python tools/time_frames.py 1000000 1920 1080 8 8 5 | grep -o "trace.*Msamples/s)"; done
for c in 0 7; do echo -n "N=16 cfg $c "; SRT_PACKET_CFG=$c python tools/time_frames.py 1000000 1920 1080 16 16 5 | grep -o "trace.*Msamples/s)"; done
echo -n "N=4 center "; python - <<'PY'
PY
python -m pytest tests -m gpu -q -x 2>&1 | tail -1
