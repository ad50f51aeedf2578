export PYTHONUNBUFFERED=1
EET_GEMV_TPC2=1 timeout 300 python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "16bit or generate or megakernel" 2>&1 | tail -1
for i in 1 2; do
timeout 200 python tools/decode_step_time.py | sed "s/^/tpc1 /"
EET_GEMV_TPC2=1 timeout 200 python tools/decode_step_time.py | sed "s/^/tpc2 /"
done
