"""SG_TRACE timeline of one call (second run): python tools/trace_call.py <prof_one args...>"""
import os
import subprocess
import sys

env = dict(os.environ, SG_TRACE="1")
r = subprocess.run([sys.executable, "tools/prof_one.py"] + sys.argv[1:], capture_output=True, text=True, env=env)
blocks = r.stderr.split("[sg trace] call total")
print("[sg trace] call total" + blocks[-1] if len(blocks) > 1 else r.stderr[-3000:])
print(r.stdout[-500:])
