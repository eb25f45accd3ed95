import subprocess, sys
for idx in (3, 7):
    for f in ("base", "noA", "noST", "noEPI"):
        try:
            r = subprocess.run([sys.executable, "scripts/probe_roles1.py", str(idx), f], capture_output=True, text=True, timeout=60)
            print(idx, f, r.stdout.strip(), r.stderr.strip()[-300:], flush=True)
        except subprocess.TimeoutExpired:
            print(idx, f, "TIMEOUT", flush=True)
