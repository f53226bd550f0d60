"""Known-answer vectors pinning the parse path.

Restated from the reference's own tests (citations inline) and from SURVEY.md
Appendix B (verified against the compiled reference, oracle/_ref).  Each entry:
(input bytes, expected code name, expected offset or None when the reference
test pins only the code).
"""

KAT = [
    # SURVEY.md App. B
    (b'["abc', "STRING_ERROR", 5),
    (b"[1,2", "TAPE_ERROR", 4),
    (b'{"a":1]', "TAPE_ERROR", 6),
    (b'[1"a"]', "NUMBER_ERROR", 1),
    (b'[true"a"]', "TAPE_ERROR", 5),
    (b"[" * 1025 + b"]" * 1025, "DEPTH_ERROR", 1024),
    (b'"\\uD834x"', "STRING_ERROR", 1),
    (b'"\\uDD1E\\uD834"', "STRING_ERROR", 1),
    (b"[1, \x01]", "TAPE_ERROR", 4),
    (b"0." + b"0" * 60 + b"1e360", "NUMBER_ERROR", 0),
    (b"0." + b"0" * 60 + b"1e300", "OK", -1),
    (b'[1,,"\xff"]', "UTF8_ERROR", 5),
    (b"[\xc3\xa9]", "TAPE_ERROR", 1),
    (b"", "EMPTY", -1),
    (b" \n", "EMPTY", -1),
    (b'"a\nb', "STRING_ERROR", 2),
    (b"[1]x", "TAPE_ERROR", 3),
    (b'{"a" "b"}', "TAPE_ERROR", 5),
    (b"[", "TAPE_ERROR", 1),
    (b'"\\', "STRING_ERROR", 1),
    (b"-", "NUMBER_ERROR", 0),
    (b"[-]", "NUMBER_ERROR", 1),
    (b"[1e400]", "NUMBER_ERROR", 1),
    (b"[1e-400]", "OK", -1),
    (b"\x00", "TAPE_ERROR", 0),
    (b'[01, "\\q"]', "NUMBER_ERROR", 1),
    (b'{"\\q":1}', "STRING_ERROR", 2),
    (b'{"a":1,"b"}', "TAPE_ERROR", 10),
    (b"\xef\xbb\xbf{}", "TAPE_ERROR", 0),
    (b"[1 2]", "TAPE_ERROR", 3),
    (b"{}}", "TAPE_ERROR", 2),
    (b"[]]", "TAPE_ERROR", 2),
    (b'{"a":[}', "TAPE_ERROR", 6),
    (b'["a\\u00"]', "STRING_ERROR", 3),
    (b"[1.]", "NUMBER_ERROR", 1),
    (b"[1.5e]", "NUMBER_ERROR", 1),
    (b"1" + b"0" * 19, "NUMBER_ERROR", 0),
    (b"-9223372036854775808", "OK", -1),
    (b'["\xed\xa0\x80"]', "UTF8_ERROR", 2),
    (b"ab\xc3", "UTF8_ERROR", 2),
    (b"\xe1\x80\x41", "UTF8_ERROR", 0),
    (b"\xc3\xa9\xa9", "UTF8_ERROR", 2),
    # proj/tests/test_tape.cpp:108-128 grammar rejections (code only)
    (b'{"a":1,}', "TAPE_ERROR", None),
    (b"[1,]", "TAPE_ERROR", None),
    (b"[12 a]", "TAPE_ERROR", None),
    (b'{"a" 1}', "TAPE_ERROR", None),
    (b'{"a":}', "TAPE_ERROR", None),
    (b"{1:2}", "TAPE_ERROR", None),
    (b'{"a":1 "b":2}', "TAPE_ERROR", None),
    (b"]", "TAPE_ERROR", None),
    (b"{", "TAPE_ERROR", None),
    (b"[1}", "TAPE_ERROR", None),
    (b"1 2", "TAPE_ERROR", None),
    (b"[] []", "TAPE_ERROR", None),
    (b"truely", "TAPE_ERROR", None),
    (b"nul", "TAPE_ERROR", None),
    (b"falsey", "TAPE_ERROR", None),
    (b",", "TAPE_ERROR", None),
    # test_tape.cpp:130-136 error kinds
    (b"   \n\t ", "EMPTY", -1),
    (b"[01]", "NUMBER_ERROR", None),
    (b'["\\q"]', "STRING_ERROR", None),
    (b'"\xed\xa0\x80"', "UTF8_ERROR", None),
    # test_tape.cpp:138-153 depth limit
    (b"[" * 1024 + b"]" * 1024, "OK", -1),
    (b'[{"k":' * 512 + b"0" + b"}]" * 512, "OK", -1),
    # test_tape.cpp:155-161 atoms
    (b"[true]", "OK", -1),
    (b"[true ]", "OK", -1),
    (b"[truex]", "TAPE_ERROR", None),
    (b'[null""]', "TAPE_ERROR", None),
    (b"true", "OK", -1),
    # test_tape.cpp:163-167 odd shapes
    (b'{"a":1,"a":2}', "OK", -1),
    (b'{"":null}', "OK", -1),
    (b'[[],{},[{}],{"a":[]}]', "OK", -1),
    # test_capi.cpp:24-41
    (b'{"a":1}', "OK", -1),
    (b'"\xff"', "UTF8_ERROR", 1),
    (b"  ", "EMPTY", -1),
    (b"7", "OK", -1),
    # test_indexer.cpp:125-132
    (b'[1, "\xb1\x87"]', "UTF8_ERROR", 5),
]

# worked example block (proj/tests/helpers.h:27-28 = PAPER.md:344) and its
# final structural row (test_bitmask.cpp:127-144)
EXAMPLE_BLOCK = b'{ "\\\\\\"Nam[{": [ 116,"\\\\\\\\" , 234, "true", false ], "t":"\\\\\\"" }'
EXAMPLE_FINAL_ROW = "1_1__________1_1_1__11______1_1__1_1_____1_1_____11_1__11______1"

# Fig. 1 document (helpers.h:31-48) and its 38-word tape (test_tape.cpp:43-73)
EXAMPLE_DOCUMENT = b"""{
\t"Width": 800,
\t"Height": 600,
\t"Title": "View from my room",
\t"Url": "http://ex.com/img.png",
\t"Private": false,
\t"Thumbnail": {
\t\t"Url": "http://ex.com/th.png",
\t\t"Height": 125,
\t\t"Width": 100
\t},
\t"array": [
\t\t116,
\t\t943,
\t\t234
\t],
\t"Owner": null
}"""
EXAMPLE_TAPE_WORDS = {0: ("r", 37), 1: ("{", 37), 15: ("{", 25), 24: ("}", 15), 26: ("[", 34),
                      33: ("]", 26), 36: ("}", 1), 37: ("r", 0)}
EXAMPLE_INTS = [(3, 800), (6, 600), (19, 125), (22, 100), (27, 116), (29, 943), (31, 234)]

# small documents with pinned indexes (test_indexer.cpp:54-71, test_capi.cpp:53-72)
INDEX_KAT = [
    (b"[12 a]", [0, 1, 4, 5]),
    (b'{"k":1}', [0, 1, 4, 5, 6]),
    (b"", []),
    (b"   \t\n  ", []),
    (b"7", [0]),
    (b"  7", [2]),
    (b'"ab"', [0]),
    (b'"a" "b"', [0, 4]),
    (b'{ "k" : [ 1 , 2 ] }', [0, 2, 6, 8, 10, 12, 14, 16, 18]),
]

SOUP_POOL = b'{}[]:,"\\\\"  \t\n0123456789abc tfn-.eE+ "\\"{}'
