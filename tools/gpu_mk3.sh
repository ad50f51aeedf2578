export PYTHONUNBUFFERED=1
EET_MK_TRACE=1 timeout 300 python tools/decode_profile.py --steps 16 2>&1 | grep -A1 "mk trace" | tail -6
