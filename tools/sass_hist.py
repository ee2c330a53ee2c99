"""Per-function SASS opcode histogram of a cubin/executable (cuobjdump -sass)."""
import collections, re, subprocess, sys

def hist(path, pattern=""):
    out = subprocess.run(["cuobjdump", "-sass", path], capture_output=True, text=True).stdout
    fn, res = None, {}
    for line in out.splitlines():
        m = re.match(r"\s+Function : (\S+)", line)
        if m:
            fn = m.group(1); res[fn] = collections.Counter(); continue
        m = re.match(r"\s+/\*[0-9a-f]+\*/\s+(@!?U?P\w+\s+)?([A-Z][A-Z0-9._]+)", line)
        if m and fn:
            res[fn][m.group(2)] += 1
    return {f: c for f, c in res.items() if re.search(pattern, f)}

if __name__ == "__main__":
    for f, c in hist(sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else "").items():
        print(f, dict(c.most_common(8)))
