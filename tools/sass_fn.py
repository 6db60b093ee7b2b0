"""Extract one function's SASS from a .so: python tools/sass_fn.py LIB SUBSTRING"""
import subprocess, sys
out = subprocess.run(["cuobjdump", "-sass", sys.argv[1]], capture_output=True, text=True).stdout
blocks = out.split("Function : ")
for b in blocks[1:]:
    name = b.split("\n", 1)[0].strip()
    if sys.argv[2] in name:
        print("Function :", b)
        break
