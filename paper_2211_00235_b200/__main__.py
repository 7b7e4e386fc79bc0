"""python -m paper_2211_00235_b200 <verify|gradcheck|bench|cost> <config>"""
import sys

from .cli import main

sys.exit(main())
