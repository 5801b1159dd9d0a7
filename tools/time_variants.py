"""Time the pricing kernel of each built variant (fresh process per variant)."""
import glob, os, subprocess, sys
root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
args = sys.argv[1:] or ["100", "20"]
for lib in sorted(glob.glob(os.path.join(root, "paper_1205_0106_b200", "_variants", "*.so"))):
    env = dict(os.environ, QMCG_LIB=lib)
    out = subprocess.run([sys.executable, os.path.join(root, "tools", "prof_price.py"), *args], env=env,
                         capture_output=True, text=True)
    print(os.path.basename(lib), out.stdout.strip(), out.stderr.strip()[-300:])
