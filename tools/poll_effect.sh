#!/bin/bash
# step time of tools/step_jitter.py alone and with an NVML poller running beside it
nproc
python - <<'PY' > /tmp/poll.py
import re
src = open("bench.py").read()
m = re.search(r'_NVML_POLL = r"""(.*?)"""', src, re.S)
open("/tmp/poll_body.py", "w").write(m.group(1))
PY
python tools/step_jitter.py 2>&1 | tail -5 | cut -c1-14
python /tmp/poll_body.py 0 > /dev/null &
P=$!
sleep 1
python tools/step_jitter.py 2>&1 | tail -5 | cut -c1-14
kill $P
sed -i 's/time.sleep(0.005)/time.sleep(0.05)/' /tmp/poll_body.py
python /tmp/poll_body.py 0 > /dev/null &
P=$!
sleep 1
python tools/step_jitter.py 2>&1 | tail -5 | cut -c1-14
kill $P
