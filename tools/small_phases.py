import sys
sys.path.insert(0,'.')
exec(open('tools/quick_phases.py').read().replace('names = ["A: P1 || chains+stop", "B1 wait", "den", "changed", "-", "P2+apply+Bcnt", "lists+B0", "-"]','names = ["B2 wait (after decision)", "den", "cand+P2+apply", "-", "publish+B1", "gather", "chains+decide", "row1 P1 gemv"]'))
