"""Print the SASS of the first function whose mangled name contains all given substrings."""
import subprocess, sys
so, pats = sys.argv[1], sys.argv[2:]
out = subprocess.run(["cuobjdump", "-sass", so], capture_output=True, text=True).stdout.splitlines()
on = False
for ln in out:
    if "Function :" in ln:
        if on:
            break
        on = all(p in ln for p in pats)
    if on:
        print(ln)
